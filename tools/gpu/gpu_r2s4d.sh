O=gpurun_out/s4d
mkdir -p $O
export CONC_MODES="2,NULPA_GROUP_STEPS=1 2,NULPA_GROUP_STEPS=4 2,NULPA_GROUP_STEPS=8"
for w in "sbm 0 20" "rmat 18 10" "rmat 22 10" "rmat 24 5" "rmat 27 3" "web 0 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
NULPA_GROUP_STEPS=8 timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_g8.log 2>&1; echo "rc=$?" >> $O/pytest_g8.log
