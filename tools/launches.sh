# Per-kernel device times of one warmed step (ncu launch list, cold-cache serialized).
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s ${1:-40} -c ${2:-24} --csv --log-file gpurun_out/launches.csv python tools/quick_time.py > /dev/null 2>&1
