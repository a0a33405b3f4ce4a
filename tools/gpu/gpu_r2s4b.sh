# Concurrent tier groups: A/B on every workload + the parity and protocol tests.
O=gpurun_out/s4b
mkdir -p $O
for w in "sbm 0 20" "rmat 16 10" "rmat 18 10" "rmat 20 10" "rmat 22 10" "rmat 24 5" "grid 0 5" "web 0 3" "rmat 27 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
NULPA_CONCURRENT=1 timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_conc1.log 2>&1; echo "rc=$?" >> $O/pytest_conc1.log
