set -x
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "not config4 and not config5" > gpurun_out/r28_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r28_pytest.log
/usr/bin/time -v timeout 1500 python bench.py > gpurun_out/r28_bench.json 2> gpurun_out/r28_bench.err; echo "bench rc=$?"
tail -25 gpurun_out/r28_bench.err | grep -i "elapsed\|maximum resident"
