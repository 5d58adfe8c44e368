# usage: bash tools/gpu_occ.sh "<cfg> <pad bytes>" ...  -- occupancy sensitivity of the DCDS kernel
for spec in "$@"; do
  set -- $spec
  out=gpurun_out/occ_$1_$2.json
  ME_SMEM_PAD=$2 timeout 300 python bench.py --config $1 --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp > $out 2>&1
  echo "$spec $(python -c "import json;d=json.load(open('$out'));print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
