O=gpurun_out/s4k
mkdir -p $O
export CONC_MODES="2 2,NULPA_GROUP_STEPS=2"
for w in "sbm 0 30" "rmat 18 10" "rmat 22 10" "rmat 27 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
