set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r36_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r36_pytest.log
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 600 python bench.py --config 4 > gpurun_out/r36_bench4.json 2> gpurun_out/r36_bench4.err; echo "bench4 rc=$?"
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r36_bench5.json 2> gpurun_out/r36_bench5.err; echo "bench5 rc=$? secs=$(( $(date +%s) - t0 ))"
timeout 900 python bench.py --impl reference > gpurun_out/r36_ref5.json 2> gpurun_out/r36_ref5.err; echo "ref rc=$?"
timeout 900 python bench.py --config 4 --ablation > gpurun_out/r36_ablation4.json 2> gpurun_out/r36_ablation4.err; echo "abl rc=$?"
