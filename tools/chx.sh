CHASE_VARIANTS=0 SKEWEIG_CHASE_DBG=1 timeout 120 python tools/chase_time.py 16384 2>&1 | tail -2
CHASE_VARIANTS=0 timeout 200 python tools/chase_time.py 32768 | tail -1
