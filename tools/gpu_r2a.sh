mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2a/tests.log
timeout 300 python tools/dump_traces.py --config c3 --pairs 1,2,3,4 --cap 48 --out gpurun_out/r2a/traces_c3.npz; echo "tr3 rc=$?"
timeout 300 python tools/dump_traces.py --config c4 --pairs 1 --cap 64 --out gpurun_out/r2a/traces_c4.npz; echo "tr4 rc=$?"
CMD="python bench.py --config c3 --steps 2 --warmup 1 --no-fs --no-e2e --no-cpu --no-cmp"
$CMD > gpurun_out/r2a/plain.json 2> gpurun_out/r2a/plain.err && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dcds_kernel -s 1 -c 1 -o gpurun_out/r2a/prof_c3 $CMD > gpurun_out/r2a/ncu.log 2>&1; echo "ncu rc=$?"
