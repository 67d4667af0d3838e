# sweep single-pass quantizer build flags on the Wan chunk (GPU box, repo root).
# usage: bash tools/sweep_quant.sh "-DKVQ_SP_THREADS=1024 -DKVQ_SP_NB=1" ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
[ -z "$NOTEST" ] && timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "quantize" 2>&1 | tail -1
for flags in "" "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
     $flags -c paper_2605_18739_b200/csrc/quant.cu -o paper_2605_18739_b200/_build/quant.cu.o > /dev/null 2>&1 || { echo "[$flags] build failed"; continue; }
  rm -f paper_2605_18739_b200/libkvq.so
  python -c "from paper_2605_18739_b200 import build as b; b.build()" > /dev/null  # re-link only (same link line)
  echo "[$flags] $(timeout 120 python tools/time_append.py 2>&1 | tail -2 | tr '\n' ' ')"
done
python -c "from paper_2605_18739_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
