set -x
nproc; lscpu | grep -i "model name"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r1_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r1_bench4.json 2> gpurun_out/r1_bench4.err; echo "bench rc=$?"
timeout 300 python scripts/quick_run.py 3 --opts 8 --reps 2 > gpurun_out/r1_q3.log 2>&1
timeout 900 python scripts/quick_run.py 5 --opts 8 --reps 1 > gpurun_out/r1_q5.log 2>&1; echo "q5 rc=$?"
