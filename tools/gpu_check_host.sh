timeout 300 python tools/host_profile.py numpy 2>&1 | head -60; timeout 300 python tools/host_profile.py sharded 2>&1 | head -60
