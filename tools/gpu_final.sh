# usage: bash tools/gpu_final.sh TAG -- what the driver runs at round end: GPU tests, smoke(), bench
TAG=${1:-final}; mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/$TAG/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/$TAG/smoke.log
timeout 900 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$TAG/ref.json 2> gpurun_out/$TAG/ref.err; echo "ref rc=$?"
