mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "modularity or quality or stats or dist" > gpurun_out/r2s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest.log
NULPA_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 24 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/r2s_gloo2.log 2>&1; tail -1 gpurun_out/r2s_gloo2.log > gpurun_out/r2s_gloo2.json
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2s_bench.json
timeout 600 python bench.py --workload web --steps 5 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2s_bench_web.json
