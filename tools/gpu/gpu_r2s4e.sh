O=gpurun_out/s4e
mkdir -p $O
timeout 900 python -m pytest tests/test_chunk_major_gpu.py -x -q > $O/pytest_cm.log 2>&1; echo "rc=$?" >> $O/pytest_cm.log
export CONC_MODES="2,NULPA_CHUNK_MAJOR=0 2"
for w in "grid 0 5" "sbm 0 20" "rmat 18 10"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --workload grid --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_grid.json
