# build attention.cu with each flag set (one per argument) and time it; GPU box, repo root
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for F in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude $F \
     -c paper_2605_18739_b200/csrc/attention.cu -o paper_2605_18739_b200/_build/attention.cu.o > /dev/null 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2605_18739_b200/libkvq.so paper_2605_18739_b200/_build/*.o -lcudart
  for rep in 1 2; do echo "[$F] $(timeout 120 python tools/quick_time.py 2>&1 | head -1)"; done
done
