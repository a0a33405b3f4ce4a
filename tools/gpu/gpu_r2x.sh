mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2x_web_launches.csv python tools/profile_run.py web 0 1 > gpurun_out/r2x_web.log 2>&1
python tools/ncu_summary.py gpurun_out/r2x_web_launches.csv > gpurun_out/r2x_web_summary.txt 2>&1
rm -f gpurun_out/r2x_web_launches.csv
