O=gpurun_out/s4f
mkdir -p $O
timeout 900 python -m pytest tests/test_chunk_major_gpu.py -x -q > $O/pytest_cm.log 2>&1; echo "rc=$?" >> $O/pytest_cm.log
export CONC_MODES="2,NULPA_CHUNK_MAJOR=0 2,NULPA_CHUNK_ROWS=1 2,NULPA_CHUNK_ROWS=2 2 2,NULPA_CHUNK_ROWS=8"
timeout 900 python tools/experiments/conc_ab.py grid 0 5 >> $O/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
