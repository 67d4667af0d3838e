#!/bin/bash
# One GPU session: tests, bench, launch list, full ncu captures.  Usage: tools/gpu_round.sh <tag> [what]
TAG=${1:-r01}; WHAT=${2:-all}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [[ $WHAT == all || $WHAT == test ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_$TAG.txt
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 8 -c 1 \
     -o gpurun_out/attn_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_attn_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_kernel|amax_kernel" -s 16 -c 2 \
     -o gpurun_out/quant_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_quant_$TAG.log 2>&1
  ls -la gpurun_out
fi
