set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r27_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r27_pytest.log
timeout 600 python bench.py > gpurun_out/r27_bench.json 2> gpurun_out/r27_bench.err; echo "bench rc=$?"
