timeout 600 python tools/byte_host_profile.py 32 2>&1 | head -45
