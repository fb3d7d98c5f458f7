for B in 32 16 64; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DNSG_FLAT_BATCH=$B -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  for st in 1 2 3 4; do
    v=$(timeout 300 python bench.py --steps 200 --warmup 10 --streams $st --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'))")
    echo "batch=$B streams=$st: $v"
  done
done
