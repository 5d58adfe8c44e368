# usage: bash tools/gpu_sweep.sh TAG CFG "ENV1;ENV2;..."  -- DCDS ms / frac of bench.py per env setting
TAG=$1; CFG=$2; IFS=';' read -ra SETS <<< "$3"
mkdir -p gpurun_out/$TAG
for e in "${SETS[@]}"; do
  n=$(echo "$e" | tr ' =,/' '____')
  env $e timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/s_${CFG}_$n.json 2> gpurun_out/$TAG/s_${CFG}_$n.err
  echo "$CFG [$e] $(python -c "import json;d=json.load(open('gpurun_out/$TAG/s_${CFG}_$n.json'));print(round(d['kernel_ms_mean'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
