mkdir -p gpurun_out/z
(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4) > gpurun_out/z/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/z/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/z/bench_c5_columns.json 2> gpurun_out/z/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/z/bench_reference_c5.json 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/z/launches_c5.csv timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"analyze_kernel|merge_kernel" -c 3 -f -o gpurun_out/z/prof_analyze_c5 timeout 900 python tools/one_launch.py c5 col 1 > gpurun_out/z/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/z/prof_analyze_c5.ncu-rep "ncu --set full --clock-control none, c5 columns, one analysis call (split: host pass 8 x 19, device pass 11 x 15, merge)" > gpurun_out/z/ncu_summary.txt 2>&1
ncu -i gpurun_out/z/prof_analyze_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/z/src_c5.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/z/src_c5.csv 40 > gpurun_out/z/ncu_lines_c5.txt 2>&1
rm -f gpurun_out/z/src_c5.csv
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize.py shard > gpurun_out/z/san_$tool.log 2>&1
done
