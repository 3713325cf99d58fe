# usage: bash tools/ncu_full.sh <kernel-regex> <out-name> [skip]
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${3:-2} -c ${4:-1} -o gpurun_out/$2 python tools/quick_time.py > gpurun_out/$2.log 2>&1
tail -3 gpurun_out/$2.log
