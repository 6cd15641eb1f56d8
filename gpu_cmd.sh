#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch list and one
# --set full capture of the two BP kernels (K5 ray_msg*, K6 tile_reduce).
#   gpurun --timeout 3000 -- 'bash gpu_cmd.sh [tests|bench|ncu|all]'
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
if [[ $what == bench || $what == all || $what == ncu ]]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1
  tail -1 gpurun_out/bench.log | cut -c1-3000
fi
if [[ $what == ncu || $what == all ]]; then
  C="python bench.py --steps 1 --warmup 1 --iters 2 --no-cpu-baseline"
  timeout 900 $C > gpurun_out/plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on \
      -k regex:'ray_msg|tile_reduce' -s 10 -c 5 -o gpurun_out/prof -f $C > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
