# ncu evidence of the current build: launch list of the C2 bench, one --set full capture of the fast kernel,
# brief captures of the next-row kernels, and the C5 sweep
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 3 -c 1 -f -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_bench.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/fast_C2_source.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_trace.csv python bench.py --path trace --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_anon.csv python bench.py --path anonymize --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_C5.json > gpurun_out/sweep.log 2>&1
