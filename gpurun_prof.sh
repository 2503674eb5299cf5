mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launch_run.log 2>&1; echo "launches=$?" >> gpurun_out/status2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:analyze_kernel -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_run.log 2>&1; echo "prof=$?" >> gpurun_out/status2.txt
