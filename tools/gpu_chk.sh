# usage: bash tools/gpu_chk.sh TAG -- GPU suite, then c3 / c4 DCDS kernel ms and c3 FS (64 pairs)
TAG=$1
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$TAG/tests.log
bash tools/gpu_dv.sh $TAG "c3 c4"
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs 64 > gpurun_out/$TAG/fs.json 2>gpurun_out/$TAG/fs.err
python -c "import json;d=json.load(open('gpurun_out/$TAG/fs.json'))['fullsearch'];print('fs c3', round(d['ms'],3), round(d['alu_frac'],3))"
