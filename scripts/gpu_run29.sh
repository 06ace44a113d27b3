set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r29_bench.json 2> gpurun_out/r29_bench.err; echo "bench rc=$? secs=$(( $(date +%s) - t0 ))"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r29_bench_ref.json 2> gpurun_out/r29_bench_ref.err; echo "ref rc=$? secs=$(( $(date +%s) - t0 ))"
for v in half wc256; do
  PBNG_CACHE=/tmp/pbng_graph_cache_r1 PBNG_TRACE=1 PBNG_LIB=paper_2110_12511_b200/libpbng_$v.so timeout 300 python scripts/quick_run.py 5 --opts 8 --reps 1 2>&1 | grep -v "^cd \|^fd " > gpurun_out/r29_${v}_5.log
done
for f in gpurun_out/r29_*_5.log; do echo $f; grep -h "tier2" $f | tail -1 | cut -c1-130; grep -h "rep" $f | tail -1 | cut -c1-200; done
