# Re-verification of the final build (profiles/r2): GPU suite, smoke, default bench, grid bench.
O=gpurun_out/${TAG:-s4j}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.log 2> $O/bench.err; tail -1 $O/bench.log > $O/bench.json
timeout 600 python bench.py --workload grid --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_grid.json
timeout 600 python bench.py --workload web --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_web.json
