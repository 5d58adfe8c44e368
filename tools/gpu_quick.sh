# usage: bash tools/gpu_quick.sh [configs...]  -- GPU tests, then DCDS ms/frac per config (20 steps)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_quick.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_quick.log
for c in "${@:-c3 c4}"; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/q_$c.json'));print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
