# compute-sanitizer passes over the GPU parity tests (memcheck + racecheck on a subset).
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 800 -k "golden or walkthrough or clustered or tiny or dense or empty or zsweep or variants or graph" 2>&1 | tail -3
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 800 -k "golden or walkthrough or clustered_long" 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_slab.py tests/test_step.py -m gpu -x -q --timeout 500 2>&1 | tail -2
timeout -s KILL 1200 compute-sanitizer --tool memcheck --print-limit 5 --target-processes all python -m pytest tests/test_modes.py -m gpu -x -q --timeout 1100 2>&1 | tail -2
