# usage: bash tools/gpu_dv.sh TAG "cfgs" v1 v2 ... -- DCDS kernel ms of libme.so and variants
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out/$TAG
for c in $CFGS; do
for v in product "$@"; do
  if [ "$v" = product ]; then LIB=""; else LIB=paper_0806_0689_b200/variants/libme_$v.so; fi
  ME_LIBRARY=$LIB timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/b_${c}_$v.json 2>gpurun_out/$TAG/b_${c}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/$TAG/b_${c}_$v.json'));print('$c $v', round(d['kernel_ms_mean'],4), round(d['roofline']['frac'],4))"
done
done
