set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r24_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r24_pytest.log
timeout 600 python bench.py > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err; echo "bench rc=$?"
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/r24_bench5.json 2> gpurun_out/r24_bench5.err; echo "bench5 rc=$?"
timeout 900 python bench.py --ablation > gpurun_out/r24_ablation.json 2> gpurun_out/r24_ablation.err; echo "abl rc=$?"
