for d in 0 1 2 3; do echo "dbg=$d"; IBC_DEBUG_SPREAD=$d timeout -s KILL 60 python tools/quick_time.py 2>&1 | tail -1; done
