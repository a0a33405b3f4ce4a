O=gpurun_out/${TAG:-s4q}
mkdir -p $O
timeout 900 python -m pytest tests/test_layout_gpu.py tests/test_dropin_cpp.py tests/test_capi.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1; do
  NULPA_STREAM_COPY=$v timeout 900 python bench.py --steps 2 --warmup 3 --e2e-steps 2 --dropin-steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > $O/bench_sc$v.json
done
