NSG_LIB_PATH_DEV=tools/libnsg_p3.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/p3_parity.txt 2>&1; echo rc $? >> gpurun_out/p3_parity.txt
out=gpurun_out/variants.txt; : > $out
for rep in 1 2; do for c in C2 U2 C3; do
  for v in tools/libnsg_*.so; do echo "== $v $c" >> $out; NSG_LIB_PATH_DEV=$v timeout 300 python tools/gpu_prof.py $c >> $out 2>&1; done
done; done
