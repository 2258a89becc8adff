timeout 300 python tools/byte_first_gate.py 32 2>&1 | head -70
