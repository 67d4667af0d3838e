# sweep the single-pass quantizer's CTA size / blocks-per-thread on the Wan chunk (GPU box, repo root)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "quantize" 2>&1 | tail -1
for cfg in "512 2" "1024 1" "768 1" "512 1" "384 2"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
     -DKVQ_QUANT_THREADS=$1 -DKVQ_QUANT_NB=$2 -c paper_2605_18739_b200/csrc/quant.cu -o paper_2605_18739_b200/_build/quant.cu.o > /dev/null 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2605_18739_b200/libkvq.so paper_2605_18739_b200/_build/*.o -lcudart
  echo "threads=$1 nb=$2 $(timeout 120 python tools/quick_time.py 2>&1 | tail -1) | $(timeout 60 python tools/trace_quant.py 2>&1 | tail -1)"
done
