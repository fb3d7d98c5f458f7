for L in 2 3; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DNSG_LANES=$L -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  echo "== lanes $L"
  timeout 600 python tools/sweep.py --min-log2 28 --max-log2 30 2>&1 | grep -o '"log2_n": [0-9]*, "dist": "[a-z]*".*"packets_per_s": [0-9.]*' | sed 's/"windows.*packets_per_s"/pps/'
done
