# lazy-rescale threshold sweep: parity tests + timing per threshold (GPU box, repo root)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in ${@:-0.0f 2.0f 8.0f}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -DKVQ_LAZY_LOG2=$L \
     -c paper_2605_18739_b200/csrc/attention.cu -o paper_2605_18739_b200/_build/attention.cu.o > /dev/null 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2605_18739_b200/libkvq.so paper_2605_18739_b200/_build/*.o -lcudart
  echo "LAZY=$L $(timeout 120 python tools/quick_time.py 2>&1 | head -1)"
  timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rollout.py -q -k "attention or w30" 2>&1 | tail -1
  timeout 120 python tools/attn_err.py 2>&1 | tail -3
done
