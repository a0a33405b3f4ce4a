mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --scale 24 --steps 2 --warmup 3 > gpurun_out/r2e_ref24.log 2> gpurun_out/r2e_ref24.err; tail -1 gpurun_out/r2e_ref24.log > gpurun_out/r2e_ref24.json
timeout 1500 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2e_ref.log 2> gpurun_out/r2e_ref.err; tail -1 gpurun_out/r2e_ref.log > gpurun_out/r2e_ref.json
