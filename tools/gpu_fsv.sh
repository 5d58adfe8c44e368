# usage: bash tools/gpu_fsv.sh TAG v1 v2 ... -- c3 FS time (64 pairs) of libme.so and variants
TAG=$1; shift
mkdir -p gpurun_out/$TAG
for v in product "$@"; do
  if [ "$v" = product ]; then LIB=""; else LIB=paper_0806_0689_b200/variants/libme_$v.so; fi
  ME_LIBRARY=$LIB timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs 64 > gpurun_out/$TAG/b_$v.json 2>gpurun_out/$TAG/b_$v.err
  python -c "import json;d=json.load(open('gpurun_out/$TAG/b_$v.json'))['fullsearch'];print('$v', round(d['ms'],3), round(d['alu_frac'],3))"
done
