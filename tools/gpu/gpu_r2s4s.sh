O=gpurun_out/s4s
mkdir -p $O
i=0
for v in 1 0 1 0; do
  i=$((i+1))
  NULPA_STREAM_COPY=$v timeout 900 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --dropin-steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > $O/bench_${i}_sc$v.json
done
