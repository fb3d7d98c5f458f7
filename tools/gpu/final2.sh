# final evidence of the build: full GPU tests, smoke, ncu (launch list + one --set full capture of the fast
# kernel + source-level stall dump), every bench line
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo rc $? >> gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo rc $? >> gpurun_out/smoke.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 3 -c 1 -f -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_bench.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/fast_C2_source.csv 2>/dev/null
ALL=1 bash tools/gpu/bench_all.sh
