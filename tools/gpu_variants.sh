# usage: bash tools/gpu_variants.sh <name>...  -- time variants/libme_<name>.so builds of the library (c3, c4)
cp paper_0806_0689_b200/libme.so /tmp/libme_base.so
for v in base "$@"; do
  if [ "$v" = base ]; then cp /tmp/libme_base.so paper_0806_0689_b200/libme.so; else cp variants/libme_$v.so paper_0806_0689_b200/libme.so; fi
  for c in c3 c4; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp > gpurun_out/var_${v}_$c.json 2>&1
    echo "$v $c $(python -c "import json;d=json.load(open('gpurun_out/var_${v}_$c.json'));print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
  done
done
cp /tmp/libme_base.so paper_0806_0689_b200/libme.so
