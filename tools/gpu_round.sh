# Round evidence: GPU tests, smoke, bench lines (ours + reference arm), launch
# list, ncu full of the top kernels, all-config timings -> gpurun_out/round/.
mkdir -p gpurun_out/round
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/round/pytest_gpu.log 2>&1; tail -2 gpurun_out/round/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round/smoke.log 2>&1; tail -1 gpurun_out/round/smoke.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/round/bench.json 2> gpurun_out/round/bench.err; tail -c 300 gpurun_out/round/bench.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/bench_ref.json 2> gpurun_out/round/bench_ref.err; tail -c 300 gpurun_out/round/bench_ref.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 20 --csv --log-file gpurun_out/round/launches.csv python tools/quick_time.py > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:^(spread_banks|interp_tma|row_sort|keys_kernel|scatter_interp)" -s 5 -c 5 -o gpurun_out/round/full python tools/quick_time.py > gpurun_out/round/ncu_full.log 2>&1; tail -1 gpurun_out/round/ncu_full.log
timeout -s KILL 900 python tools/config_time.py c1 c2 w128 rbc clustered severe > gpurun_out/round/configs.txt 2>&1; tail -12 gpurun_out/round/configs.txt
timeout -s KILL 600 python bench.py --workload w256 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/round/bench_w256.json 2> gpurun_out/round/bench_w256.err; tail -c 200 gpurun_out/round/bench_w256.json
