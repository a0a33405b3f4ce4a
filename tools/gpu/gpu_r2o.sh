mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_pytest.log
for k in 1 2 3 4 5 6; do timeout 120 python -m pytest tests/test_parity_gpu.py -q -k "disjoint or two_triangles or team_hub" 2>&1 | tail -1; done > gpurun_out/r2o_kat.log
bash tools/ab_env.sh rolow NULPA_RO_LOW "0 1" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2o_ab.txt 2>&1
bash tools/ab_env.sh rolowweb NULPA_RO_LOW "0 1" --workload web --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2o_ab.txt 2>&1
bash tools/ab_env.sh rolowsbm NULPA_RO_LOW "0 1" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2o_ab.txt 2>&1
bash tools/ab_env.sh rolowgrid NULPA_RO_LOW "0 1" --workload grid --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2o_ab.txt 2>&1
