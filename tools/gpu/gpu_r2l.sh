mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.log
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_w1024.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2l_ab.txt 2>&1
for w in sbm grid web; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2l_bench_$w.json
done
timeout 900 python bench.py --scale 24 --steps 5 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2l_bench_rmat24.json
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2l_ref.log 2> gpurun_out/r2l_ref.err; tail -1 gpurun_out/r2l_ref.log > gpurun_out/r2l_ref.json
