# usage: bash tools/gpu_tune.sh "<cfg> <G> <tile> [NW]" ...
set +x
for spec in "$@"; do
  set -- $spec
  NW=${4:-4}
  out=gpurun_out/tune_$1_$2_$3_$NW.json
  ME_NW=$NW ME_G=$2 ME_TILE=$3 timeout 300 python bench.py --config $1 --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp > $out 2>&1
  echo "$spec $(python -c "import json;d=json.load(open('$out'));print(round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['frac'],4), d['roofline']['bound'])" 2>&1 | tail -1)"
done
