# sweep attention build flags (GPU box, repo root): bash tools/sweep_attn_flags.sh "-DKVQ_COMBINE_SPLIT=8" ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for flags in "" "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude $flags \
     -c paper_2605_18739_b200/csrc/attention.cu -o paper_2605_18739_b200/_build/attention.cu.o > /dev/null 2>&1 || { echo "[$flags] build failed"; continue; }
  rm -f paper_2605_18739_b200/libkvq.so
  python -c "from paper_2605_18739_b200 import build as b; b.build()" > /dev/null  # re-link only (same link line)
  echo "[$flags]"; timeout 120 python tools/attn_timing.py 2>&1 | tail -5
done
python -c "from paper_2605_18739_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
