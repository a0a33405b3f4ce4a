mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2g_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g_bench.log 2> gpurun_out/r2g_bench.err; tail -1 gpurun_out/r2g_bench.log > gpurun_out/r2g_bench.json
for w in sbm grid web; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2g_bench_$w.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2g_launches_bench.log 2>&1
