# time every tools/libnsg_*.so variant against the product build on C2 (and U2): gpu_prof timing lines
out=gpurun_out/variants.txt; : > $out
for c in ${CFGS:-C2}; do
  echo "== base $c" >> $out; timeout 300 python tools/gpu_prof.py $c >> $out 2>&1
  for v in tools/libnsg_*.so; do echo "== $v $c" >> $out; NSG_LIB_PATH_DEV=$v timeout 300 python tools/gpu_prof.py $c >> $out 2>&1; done
done
