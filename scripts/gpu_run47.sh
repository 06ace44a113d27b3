set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "components" > gpurun_out/r47_pytest_lvl.log 2>&1; echo "pytest lvl rc=$?"
tail -3 gpurun_out/r47_pytest_lvl.log
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 600 python scripts/level_run.py 3 --oracle-frac 0.002 > gpurun_out/r47_level_3.log 2>&1; echo "level 3 rc=$?"
timeout 600 python scripts/level_run.py 4 --oracle-frac 0.0002 > gpurun_out/r47_level_4.log 2>&1; echo "level 4 rc=$?"
timeout 900 python scripts/level_run.py 5 --reps 1 > gpurun_out/r47_level_5.log 2>&1; echo "level 5 rc=$?"
cat gpurun_out/r47_level_*.log | grep '^{'
