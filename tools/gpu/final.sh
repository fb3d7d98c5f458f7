# full GPU test suite, smoke, every bench line, trace/anonymize launch summaries
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo rc $? >> gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo rc $? >> gpurun_out/smoke.txt
ALL=1 bash tools/gpu/bench_all.sh
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_trace.csv python bench.py --path trace --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_anon.csv python bench.py --path anonymize --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python tools/trace_time.py > gpurun_out/trace_time.txt 2>&1
