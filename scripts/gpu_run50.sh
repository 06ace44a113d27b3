set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config5 or config4" > gpurun_out/r50_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r50_pytest.log
