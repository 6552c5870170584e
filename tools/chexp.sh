n=${N:-16384}
CHASE_VARIANTS=0 SKEWEIG_CHASE_DBG=1 timeout 120 python tools/chase_time.py $n 2>&1 | tail -3
