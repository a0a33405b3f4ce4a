# Session-4 re-entry check: GPU suite + smoke on the restored build, SBM launch list.
mkdir -p gpurun_out
O=gpurun_out/s4a
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 300 python tools/experiments/sbm_profile.py > $O/sbm_profile.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_sbm.csv python tools/experiments/sbm_profile.py > $O/ncu_sbm.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --dropin-steps 0 --no-cpu-baseline > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
