# usage: bash tools/gpu_fssw2.sh TAG CFG "ENV ..." -- FS (32 pairs) of CFG per environment setting
TAG=$1; mkdir -p gpurun_out/$TAG
for e in $3; do
  n=$(echo "$e" | tr ' =,/:' '_____')
  env $(echo $e | tr ':' ' ') timeout 300 python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/fs_$2_$n.json 2>/dev/null
  echo "$2 [$e] $(python -c "import json;d=json.load(open('gpurun_out/$TAG/fs_$2_$n.json'))['fullsearch'];print(round(d['ms'],4), round(d['alu_frac'],4))" 2>&1 | tail -1)"
done
