O=gpurun_out/s4i
mkdir -p $O
CONC_MODES="2 2,NULPA_CHUNK_ROWS=24 2,NULPA_CHUNK_ROWS=28" timeout 900 python tools/experiments/conc_ab.py grid 0 5 >> $O/ab.txt 2>&1
export CONC_MODES="2 5"
for w in "rmat 27 5" "rmat 24 5" "web 0 3"; do
  timeout 900 python tools/experiments/conc_ab.py $w >> $O/ab.txt 2>&1
done
NULPA_CONCURRENT=5 timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
