mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; df -h /dev/shm /tmp; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/r2b_box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/r2b_bench.log 2>&1; tail -1 gpurun_out/r2b_bench.log > gpurun_out/r2b_bench.json
