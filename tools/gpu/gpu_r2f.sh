mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_smoke.log
bash tools/ab_env.sh grp NULPA_GROUP_STEPS "1 4 8" --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2f_ab.txt 2>&1
bash tools/ab_env.sh pair NULPA_THREAD_PAIR "0 1" --steps 5 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/r2f_ab.txt 2>&1
bash tools/ab_env.sh sbmbatch NULPA_BATCH_PASSES "1 4 20" --workload sbm --steps 20 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/r2f_ab.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2f_bench.log 2> gpurun_out/r2f_bench.err; tail -1 gpurun_out/r2f_bench.log > gpurun_out/r2f_bench.json
