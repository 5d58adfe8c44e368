# usage: bash tools/gpu_env.sh TAG "cfgs" "ENV ..." -- DCDS kernel ms per environment setting
# (ENV items: VAR=V[:VAR2=V2]; X=1 = defaults)
TAG=$1; mkdir -p gpurun_out/$TAG
for c in $2; do
for e in $3; do
  n=$(echo "$e" | tr ' =,/:' '_____')
  env $(echo $e | tr ':' ' ') timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/b_${c}_$n.json 2>/dev/null
  echo "$c [$e] $(python -c "import json;d=json.load(open('gpurun_out/$TAG/b_${c}_$n.json'));print(round(d['kernel_ms_mean'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
done
