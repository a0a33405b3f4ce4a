mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_pytest.log
for w in rmat sbm web; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2u_bench_$w.json
done
