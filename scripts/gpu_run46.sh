set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r46_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r46_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r46_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r46_smoke.log
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r46_bench5.json 2> gpurun_out/r46_bench5.err; echo "bench5 rc=$? secs=$(( $(date +%s) - t0 ))"
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 600 python bench.py --config 4 > gpurun_out/r46_bench4.json 2> gpurun_out/r46_bench4.err; echo "bench4 rc=$?"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r46_ref5.json 2> gpurun_out/r46_ref5.err; echo "ref rc=$? secs=$(( $(date +%s) - t0 ))"
