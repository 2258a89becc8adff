timeout 300 python tools/cold_probe.py 33
timeout 300 python tools/cold_probe.py 33
timeout 300 python tools/cold_probe.py 33
