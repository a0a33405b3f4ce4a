mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dist_gloo.py -x -q > gpurun_out/r2e_dist.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_dist.log
NULPA_BENCH_GLOO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 22 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/r2e_gloo2.log 2>&1; tail -1 gpurun_out/r2e_gloo2.log > gpurun_out/r2e_gloo2.json
timeout 600 python bench.py --impl reference --scale 24 --steps 2 --warmup 3 > gpurun_out/r2e_ref24.log 2> gpurun_out/r2e_ref24.err; tail -1 gpurun_out/r2e_ref24.log > gpurun_out/r2e_ref24.json
timeout 1500 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2e_ref.log 2> gpurun_out/r2e_ref.err; tail -1 gpurun_out/r2e_ref.log > gpurun_out/r2e_ref.json
