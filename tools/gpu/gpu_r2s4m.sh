# Launch list + ncu --set full tier captures of the final build (profiles/r2).
O=gpurun_out/s4m
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_r27.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:"k_(thread|group|team|wide|cluster|hub_accum)" -c 60 \
  -o $O/tiers python tools/profile_run.py 27 0 1 > $O/ncu_tiers.log 2>&1
python tools/ncu_traffic.py $O/tiers.ncu-rep > $O/ncu_traffic_r27.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_mod" -c 10 -o $O/k7 python tools/profile_k7.py 27 > $O/ncu_k7.log 2>&1
python tools/ncu_summary.py $O/launches_r27.csv $O/tiers.ncu-rep $O/k7.ncu-rep > $O/ncu_summary_r27.txt 2>&1
rm -f $O/tiers.ncu-rep $O/k7.ncu-rep
timeout 600 ncu --set full --clock-control none -k regex:"k_chunk_walk" -s 3 -c 1 \
  -o $O/grid_chunk python tools/profile_run.py grid 0 1 > $O/ncu_grid_chunk.log 2>&1
python - $O > $O/ncu_grid_final.txt 2>&1 <<'PY'
import sys
sys.path.insert(0, "tools")
import ncu_summary as S
S.full(f"{sys.argv[1]}/grid_chunk.ncu-rep")
PY
rm -f $O/grid_chunk.ncu-rep
