mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_parity_gpu.py tests/test_bench_gpu.py -m gpu -x -q > gpurun_out/r2b/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b/tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cmp --cpu-seconds 3 > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cmp --no-cpu --no-fs --scaling strong > gpurun_out/r2b/bench_strong.json 2> gpurun_out/r2b/bench_strong.err; echo "bench strong rc=$?"
