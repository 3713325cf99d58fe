for d in 15 23; do echo "dbg=$d"; IBC_DEBUG_INTERP=$d timeout -s KILL 30 python tools/quick_time.py 2>&1 | tail -1; done
