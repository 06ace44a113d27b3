set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r30_plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r30_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r30_ncu_list.log 2>&1
echo "ncu list rc=$?"
