O=gpurun_out/s4c
mkdir -p $O
export CONC_MODES="2,NULPA_SMALL_TIER_BATCH=0 2"
for w in "sbm 0 20" "rmat 16 10" "rmat 18 10" "rmat 20 10"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
export CONC_MODES="0 3 4"
for w in "rmat 24 5" "rmat 27 3" "web 0 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
