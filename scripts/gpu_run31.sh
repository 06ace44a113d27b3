set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "not config4 and not config5" > gpurun_out/r31_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r31_pytest.log
timeout 200 python scripts/quick_run.py 3 --opts 8 --reps 2 > gpurun_out/r31_q3.log 2>&1
PBNG_TRACE=1 timeout 200 python scripts/quick_run.py 4 --opts 8 --reps 2 > gpurun_out/r31_q4.log 2>&1
PBNG_TRACE=1 PBNG_CACHE=/tmp/pbng_graph_cache_r1 timeout 400 python scripts/quick_run.py 5 --opts 8 --reps 1 > gpurun_out/r31_q5.log 2>&1; echo "q5 rc=$?"
