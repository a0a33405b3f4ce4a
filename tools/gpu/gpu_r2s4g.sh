O=gpurun_out/s4g
mkdir -p $O
export CONC_MODES="2 2,NULPA_CHUNK_ROWS=14 2,NULPA_CHUNK_ROWS=8 2,NULPA_CHUNK_ROWS=18"
timeout 900 python tools/experiments/conc_ab.py grid 0 5 >> $O/ab.txt 2>&1
