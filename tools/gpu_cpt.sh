# usage: bash tools/gpu_cpt.sh TAG [full] -- compact-set tests (product + ME_DEBUG build), c4 / c3
# bench with the compact set on (default) and off (ME_COMPACT=0), the overflow kernels' ncu
# launch list; with "full" the whole GPU suite
TAG=$1
mkdir -p gpurun_out/$TAG
timeout 400 python -m pytest tests/test_compact_gpu.py tests/test_debug_build_gpu.py -x -q > gpurun_out/$TAG/compact.log 2>&1; echo "compact rc=$?"; tail -3 gpurun_out/$TAG/compact.log
for c in c4 c3; do
  for m in default 0; do
    if [ $m = default ]; then unset ME_COMPACT; else export ME_COMPACT=$m; fi
    timeout 150 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/b_${c}_$m.json 2> gpurun_out/$TAG/b_${c}_$m.err
    echo "$c compact=$m $(python -c "import json;d=json.load(open('gpurun_out/$TAG/b_${c}_$m.json'));print(round(d['kernel_ms_mean'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d.get('gpu_launches'))" 2>&1 | tail -1)"
  done
done
unset ME_COMPACT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dcds --csv --log-file gpurun_out/$TAG/ncu_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/ncu.log 2>&1
grep gpu__time_duration gpurun_out/$TAG/ncu_c4.csv | awk -F'","' '{print $5" "$NF}' | tail -4
if [ "$2" = full ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$TAG/tests.log
fi
