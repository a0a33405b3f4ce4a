O=gpurun_out/s4n
mkdir -p $O
export CONC_MODES="2 2,NULPA_CHUNK_TPS=1536,NULPA_CHUNK_ROWS=34 2,NULPA_CHUNK_TPS=1536,NULPA_CHUNK_ROWS=32 2,NULPA_CHUNK_TPS=1024,NULPA_CHUNK_ROWS=34"
timeout 900 python tools/experiments/conc_ab.py grid 0 5 >> $O/ab.txt 2>&1
