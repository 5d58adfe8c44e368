mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_bench_gpu.py -m gpu -x -q > gpurun_out/r2c/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2c/tests.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int_peaks tools/int_peaks.cu && timeout 300 /tmp/int_peaks > gpurun_out/r2c/int_peaks.json; echo "int_peaks rc=$?"
timeout 600 python tools/series.py --outdir gpurun_out/r2c > gpurun_out/r2c/series.log 2>&1; echo "series rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cmp --cpu-seconds 3 > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err; echo "bench rc=$?"
CMD="python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu --no-cmp --no-mcsse"
$CMD > gpurun_out/r2c/c4plain.json 2> gpurun_out/r2c/c4plain.err && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs_kernel -s 1 -c 1 -o gpurun_out/r2c/prof_fs_c4 $CMD > gpurun_out/r2c/ncu_fs.log 2>&1; echo "ncu fs rc=$?"
