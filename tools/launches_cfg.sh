# Launch list (ncu, cold/serialized) of one warmed step of a config_time workload.
# usage: bash tools/launches_cfg.sh <config> [skip] [count]
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s ${2:-40} -c ${3:-14} --csv --log-file gpurun_out/launches_$1.csv python tools/config_time.py $1 > /dev/null 2>&1
