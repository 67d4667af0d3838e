# timing experiments on the attention kernel (GPU box, repo root): each line rebuilds attention.cu with flags
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() {
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude $2 \
     -c paper_2605_18739_b200/csrc/attention.cu -o paper_2605_18739_b200/_build/attention.cu.o > /dev/null 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2605_18739_b200/libkvq.so paper_2605_18739_b200/_build/*.o -lcudart
  echo "$1: $(timeout 120 python tools/quick_time.py 2>&1 | head -1)"
}
if [ $# -gt 0 ]; then for f in "$@"; do run "$f" "$f"; done; exit 0; fi
run base ""
run no_max "-DKVQ_EXPERIMENT_NO_MAX"
run no_sum "-DKVQ_EXPERIMENT_NO_SUM"
run no_rescale "-DKVQ_EXPERIMENT_NO_RESCALE"
run no_all "-DKVQ_EXPERIMENT_NO_MAX -DKVQ_EXPERIMENT_NO_SUM -DKVQ_EXPERIMENT_NO_RESCALE"
