# usage: bash tools/gpu_ab.sh TAG "c3 c4" variant1 variant2 ...  -- GPU test suite on libme.so,
# then bench DCDS ms / roofline frac of libme.so and of each variants/libme_<v>.so
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$TAG/tests.log
for c in $CFGS; do
  for v in product "$@"; do
    if [ "$v" = product ]; then LIB=""; else LIB=paper_0806_0689_b200/variants/libme_$v.so; fi
    ME_LIBRARY=$LIB timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/b_${c}_$v.json 2> gpurun_out/$TAG/b_${c}_$v.err
    echo "$c $v $(python -c "import json;d=json.load(open('gpurun_out/$TAG/b_${c}_$v.json'));print(round(d['kernel_ms_mean'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
  done
done
