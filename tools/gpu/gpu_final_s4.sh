# Round-2 final evidence on the last build (profiles/<TAG>/): tools/gpu/gpu_final.sh plus the
# chunk-major grid captures. usage: tools/gpu/gpu_final_s4.sh TAG
TAG=${1:-r2}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.log 2> $O/bench.err; tail -1 $O/bench.log > $O/bench.json
for w in sbm grid web; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_$w.json
done
timeout 900 python bench.py --scale 24 --steps 5 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_rmat24.json
timeout 1500 python bench.py --impl reference > $O/bench_reference.log 2> $O/bench_reference.err; tail -1 $O/bench_reference.log > $O/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_r27.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:"k_(thread|group|team|wide|cluster|hub_accum)" -c 60 \
  -o $O/tiers python tools/profile_run.py 27 0 1 > $O/ncu_tiers.log 2>&1
python tools/ncu_traffic.py $O/tiers.ncu-rep > $O/ncu_traffic_r27.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_mod" -c 10 -o $O/k7 python tools/profile_k7.py 27 > $O/ncu_k7.log 2>&1
python tools/ncu_summary.py $O/launches_r27.csv $O/tiers.ncu-rep $O/k7.ncu-rep > $O/ncu_summary_r27.txt 2>&1
rm -f $O/tiers.ncu-rep $O/k7.ncu-rep
# the grid's thread tier, pass 3: the bucket-order chunk walk against the chunk-major one
NULPA_CHUNK_MAJOR=0 timeout 600 ncu --set full --clock-control none -k regex:"k_thread" -s 3 -c 1 \
  -o $O/grid_bucket python tools/profile_run.py grid 0 1 > $O/ncu_grid_bucket.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_chunk_walk" -s 3 -c 1 \
  -o $O/grid_chunk python tools/profile_run.py grid 0 1 > $O/ncu_grid_chunk.log 2>&1
python - $O > $O/ncu_grid.txt 2>&1 <<'PY'
import sys
sys.path.insert(0, "tools")
import ncu_summary as S
o = sys.argv[1]
for tag in ("grid_bucket", "grid_chunk"):
    print(f"== {tag}")
    S.full(f"{o}/{tag}.ncu-rep")
PY
rm -f $O/grid_bucket.ncu-rep $O/grid_chunk.ncu-rep
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_parity_gpu.py tests/test_chunk_major_gpu.py -q -x -k "sync_step or trajectory or chunk_major_layout or gates_match" > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
