# anonymiser evidence (f2): smoke, anon parity tests, anon bench line + per-kernel launch list -> gpurun_out/anon/
set -u
mkdir -p gpurun_out/anon
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc=$? >> gpurun_out/smoke.txt
timeout 400 python -m pytest tests/test_gpu_anon.py -x -q > gpurun_out/anon/tests.log 2>&1; tail -2 gpurun_out/anon/tests.log
timeout 300 python bench.py --path anonymize --steps 50 --warmup 10 > gpurun_out/anon/bench.json 2> gpurun_out/anon/bench.err; tail -c 300 gpurun_out/anon/bench.json
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 60 --csv --log-file gpurun_out/anon/launches.csv python bench.py --path anonymize --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
