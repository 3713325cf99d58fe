# compute-sanitizer passes over the GPU parity tests (memcheck + racecheck on a subset).
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 800 -k "golden or walkthrough or clustered or tiny or dense or empty or zsweep or variants or graph or concurrent" 2>&1 | tail -3
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 800 -k "golden or walkthrough or clustered_long" 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_step.py -m gpu -x -q --timeout 500 2>&1 | tail -2
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q --timeout 800 -k "golden or peskin4 or counts or (radix and 2)" 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity_configs.py -m gpu -x -q --timeout 500 -k "tma_gather and 64" 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 tests/cpp/build/slab_test 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 tests/cpp/build/overlay_test verify 2>&1 | tail -2
timeout -s KILL 1200 compute-sanitizer --tool memcheck --print-limit 5 --target-processes all python -m pytest tests/test_modes.py -m gpu -x -q --timeout 1100 2>&1 | tail -2
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_f32.py -m gpu -x -q --timeout 500 -k "not config2" 2>&1 | tail -2
