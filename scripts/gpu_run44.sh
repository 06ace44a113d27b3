set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "components" > gpurun_out/r44_pytest_lvl.log 2>&1; echo "pytest lvl rc=$?"
tail -3 gpurun_out/r44_pytest_lvl.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not config4 and not config5 and not components" > gpurun_out/r44_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r44_pytest.log
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
for c in 3 4 5; do
  timeout 600 python scripts/level_run.py $c > gpurun_out/r44_level_$c.log 2>&1; echo "level $c rc=$?"
done
cat gpurun_out/r44_level_*.log | grep '^{'
