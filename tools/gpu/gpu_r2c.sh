mkdir -p gpurun_out
date +%s > gpurun_out/r2c_times.txt
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2c_ref.log 2> gpurun_out/r2c_ref.err; tail -1 gpurun_out/r2c_ref.log > gpurun_out/r2c_ref.json
date +%s >> gpurun_out/r2c_times.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c_bench.log 2> gpurun_out/r2c_bench.err; tail -1 gpurun_out/r2c_bench.log > gpurun_out/r2c_bench.json
date +%s >> gpurun_out/r2c_times.txt
