#!/bin/bash
# One GPU session: tests, bench, launch list, full ncu captures.  Usage: tools/gpu_round.sh <tag> [all|test|bench|ncu]
TAG=${1:-r02}; WHAT=${2:-all}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build_$TAG.log; exit 1; }
if [[ $WHAT == all || $WHAT == test ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -30 | tee gpurun_out/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke_$TAG.txt
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py 2>gpurun_out/bench_$TAG.err | tail -1 | tee gpurun_out/bench_$TAG.json
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_ref_$TAG.json
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
     python bench.py --steps 3 --warmup 3 --no-cpu --no-rollout --sustain-s 0.05 > gpurun_out/ncu_bench_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ws -s 8 -c 1 \
     -o gpurun_out/attn_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu --no-rollout --sustain-s 0.05 > gpurun_out/ncu_attn_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant -s 8 -c 1 \
     -o gpurun_out/quant_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu --no-rollout --sustain-s 0.05 > gpurun_out/ncu_quant_$TAG.log 2>&1
  ls gpurun_out | grep $TAG
fi
