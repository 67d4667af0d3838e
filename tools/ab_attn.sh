#!/bin/bash
# A/B timing of attention.cu variants on the GPU box (development aid; bench.py is the contract).
# usage: bash tools/ab_attn.sh <rounds> "<src.cu> [nvcc flags]" ...   ("." = the tree's attention.cu)
# TOOL=tools/trace_attn.py prints the CTA-0 timeline of each variant instead of the timings.
ROUNDS=$1; shift
VARIANTS=("$@")
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq 1 $ROUNDS); do
  for v in "${VARIANTS[@]}"; do
    read -r src flags <<< "$v"
    [[ $src == . ]] && src=paper_2605_18739_b200/csrc/attention.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude \
       -Ipaper_2605_18739_b200/csrc $flags -c $src -o paper_2605_18739_b200/_build/attention.cu.o > /tmp/ab_build.log 2>&1 \
       || { echo "[$v] build failed"; tail -3 /tmp/ab_build.log; continue; }
    rm -f paper_2605_18739_b200/libkvq.so
    python -c "from paper_2605_18739_b200 import build as b; b.build()" > /dev/null
    if [[ -n $TOOL ]]; then echo "[round $r: $v]"; timeout 120 python $TOOL 2>&1 | tail -8
    else echo "[round $r: $v] $(timeout 120 python tools/attn_timing.py 2>&1 | grep -E 'graph|zero-fill' | tr '\n' ' ')"; fi
  done
done
python -c "from paper_2605_18739_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
