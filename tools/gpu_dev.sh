# Dev loop on the GPU: parity tests (fail fast) + timing probe.
timeout -s KILL 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 200 python tools/quick_time.py 2>&1 | tail -4
