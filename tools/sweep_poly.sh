# sweep the MUFU/FMA exp2 split (KVQ_POLY_PAIRS of 8) on the Wan layer; run from the repo root on the GPU box
set -e
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or bf16kv" 2>&1 | tail -1
for P in ${@:-0 1 2 3}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -DKVQ_POLY_PAIRS=$P \
     -c paper_2605_18739_b200/csrc/attention.cu -o paper_2605_18739_b200/_build/attention.cu.o > /dev/null 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2605_18739_b200/libkvq.so paper_2605_18739_b200/_build/*.o -lcudart
  echo "POLY_PAIRS=$P $(timeout 120 python tools/quick_time.py 2>&1 | head -1)"
done
