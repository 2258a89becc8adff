"""CPU stand-in for distributed.CudaBackend — TEST ONLY.

Lets the multi-rank control plane (remap planner, swap choreography,
measurement reductions, reference ledgers) run as real processes over gloo
on a machine without GPUs.  The arithmetic is the oracle's numpy kernels;
peer memory is emulated with torch.distributed send/recv of whole slices.
"""
import numpy as np
import torch

from oracle import ref_kernels
from paper_2511_03359_b200 import _native as nat


class NumpyBackend:
    def __init__(self, dist, n_local, mode):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.n_local = n_local
        self.psi = np.zeros(1 << n_local, dtype=np.complex128)
        if self.rank == 0:
            self.psi[0] = 1.0
        self.link_bytes = 0
        self.bpe = mode.bytes_per_element

    def apply_local(self, ops):
        for op in ops:
            m = np.array(op.m[:32])
            if op.kind == nat.SV_OP_1Q:
                ref_kernels.gate1(self.psi, op.qa, m[:8].view(np.complex128).reshape(2, 2))
            elif op.kind == nat.SV_OP_2Q:
                ref_kernels.gate2(self.psi, op.qa, op.qb, m.view(np.complex128).reshape(4, 4))
            else:
                bits = tuple(b for b in range(self.n_local) if (op.diag_mask >> b) & 1)
                ref_kernels.diag(self.psi, bits, complex(m[0], m[1]))

    def _exchange(self, partner):
        mine = torch.from_numpy(self.psi.view(np.float64).copy())
        theirs = torch.empty_like(mine)
        if self.rank < partner:
            self.dist.send(mine, partner)
            self.dist.recv(theirs, partner)
        else:
            self.dist.recv(theirs, partner)
            self.dist.send(mine, partner)
        return theirs.numpy().view(np.complex128)

    def swap(self, global_pos, local_pos):
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        side = (self.rank >> bit) & 1
        other = self._exchange(partner)
        idx = np.arange(self.psi.size)
        sel = ((idx >> local_pos) & 1) == 1 - side
        self.psi[sel] = other[idx[sel] ^ (1 << local_pos)]
        self.link_bytes += (self.psi.size // 2) * self.bpe

    def swap_group(self, pairs):
        # the same exchange as k sequential pairwise swaps (disjoint bit pairs)
        for gp, lp in pairs:
            self.swap(gp, lp)

    def swap_then_apply(self, pairs, ops, before=()):
        if before:
            self.apply_local(list(before))
        for gp, lp in pairs:
            self.swap(gp, lp)
        if ops:
            self.apply_local(ops)

    def measure_local(self):
        n = self.n_local
        norm = float(np.real(np.vdot(self.psi, self.psi)))
        ones = np.zeros(n)
        cross = np.zeros(n, dtype=np.complex128)
        for q in range(n):
            v = self.psi.reshape(-1, 2, 1 << q)
            ones[q] = float(np.sum(np.abs(v[:, 1, :]) ** 2))
            cross[q] = complex(np.sum(v[:, 0, :].conj() * v[:, 1, :]))
        return norm, ones, cross

    def pair_dot(self, global_pos):
        bit = global_pos - self.n_local
        partner = self.rank ^ (1 << bit)
        other = self._exchange(partner)
        half = self.psi.size // 2
        if (self.rank >> bit) & 1 == 0:
            a0, a1 = self.psi[:half], other[:half]
        else:
            a0, a1 = other[half:], self.psi[half:]
        return complex(np.sum(a0.conj() * a1))

    def export(self):
        return self.psi.copy()
