set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r15_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r15_pytest.log
timeout 600 python bench.py > gpurun_out/r15_bench.json 2> gpurun_out/r15_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r15_bench_ref.json 2> gpurun_out/r15_bench_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r15_plain_b.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r15_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r15_ncu_list.log 2>&1
echo "ncu list rc=$?"
