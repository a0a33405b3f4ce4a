O=gpurun_out/s4o
mkdir -p $O
export CONC_MODES="2,NULPA_FORK_BASE=0 2"
for w in "sbm 0 30" "rmat 18 10" "rmat 22 10" "rmat 27 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
