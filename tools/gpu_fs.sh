# usage: bash tools/gpu_fs.sh TAG  -- FS parity tests, then FS timing at c3 / c4 (bench's fullsearch leg)
TAG=$1; mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -x -q -k "fs or full or FS" > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$TAG/tests.log
for c in c3 c4; do
  for e in "X=1" "${@:2}"; do
    n=$(echo "$e" | tr ' =,/' '____')
    env $e timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/fs_${c}_$n.json 2> gpurun_out/$TAG/fs_${c}_$n.err
    echo "$c [$e] $(python -c "import json;d=json.load(open('gpurun_out/$TAG/fs_${c}_$n.json'))['fullsearch'];print(round(d['ms'],4), round(d['alu_frac'],4))" 2>&1 | tail -1)"
  done
done
