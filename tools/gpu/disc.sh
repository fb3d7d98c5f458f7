NSG_LIB_PATH_DEV=tools/libnsg_disc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_weighted.py -x -q > gpurun_out/d_parity.txt 2>&1; echo rc $? >> gpurun_out/d_parity.txt
out=gpurun_out/variants.txt; : > $out
for c in C2 U2 C3; do
  for v in tools/libnsg_*.so; do echo "== $v $c" >> $out; NSG_LIB_PATH_DEV=$v timeout 300 python tools/gpu_prof.py $c >> $out 2>&1; done
done
for v in base disc; do
  NSG_LIB_PATH_DEV=tools/libnsg_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fast_kernel -s 3 -c 3 --csv --log-file gpurun_out/dram_$v.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
