set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r49_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r49_smoke.log
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r49_bench5.json 2> gpurun_out/r49_bench5.err; echo "bench5 rc=$? secs=$(( $(date +%s) - t0 ))"
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 600 python bench.py --config 4 > gpurun_out/r49_bench4.json 2> gpurun_out/r49_bench4.err; echo "bench4 rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "components or tiny_corpus or config3_parity" > gpurun_out/r49_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r49_pytest.log
