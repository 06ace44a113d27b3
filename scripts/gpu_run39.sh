set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r39_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r39_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r39_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/r39_smoke.log | tail -2
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r39_bench5.json 2> gpurun_out/r39_bench5.err; echo "bench5 rc=$? secs=$(( $(date +%s) - t0 ))"
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 600 python bench.py --config 4 > gpurun_out/r39_bench4.json 2> gpurun_out/r39_bench4.err; echo "bench4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r39_ref5.json 2> gpurun_out/r39_ref5.err; echo "ref rc=$?"
timeout 300 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r39_plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r39_launches4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r39_ncu.log 2>&1
echo "ncu rc=$?"
