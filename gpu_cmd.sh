#!/bin/bash
# One gpurun call: GPU parity tests + smoke, the default bench line, the ncu launch list, the
# per-launch DRAM traffic of one BP iteration (K5 classes + K6) and one --set full capture of the
# largest K5 class kernel and of K6 / K6b; "modes": every mode's bench line.
#   gpurun --timeout 3000 -- 'bash gpu_cmd.sh [tests|bench|ncu|modes|all]'
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
fi
if [[ $what == bench || $what == all || $what == ncu ]]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1
  tail -1 gpurun_out/bench.log | cut -c1-400
fi
if [[ $what == ncu || $what == all ]]; then
  C="python bench.py --steps 1 --warmup 1 --iters 2 --no-cpu-baseline"
  timeout 900 $C > gpurun_out/plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:'ray_msg|tile_reduce|block_reduce' -o gpurun_out/traffic -f $C > gpurun_out/ncu_traffic.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:'ray_msg_kernel<\(int\)16, \(int\)6|tile_reduce|block_reduce' -s 2 -c 2 -o gpurun_out/prof -f $C > gpurun_out/ncu_full.log 2>&1
  tail -1 gpurun_out/ncu_full.log; du -sh gpurun_out
fi
if [[ $what == modes || $what == all ]]; then
  # every mode's bench line (frames30 unless named), and the 0.02 m config on 4 emulated ranks
  for m in "sparse:--bricks 8" "patch:--noise patch" "kfavg:--messages keyframe-avg" "mf:--matrix-free 5" "frames100:--config frames100 --steps 2 --warmup 3"; do
    n=${m%%:*}; a=${m#*:}
    timeout 900 python bench.py --no-cpu-baseline $a > gpurun_out/bench_$n.log 2>&1
    echo "$n $(tail -1 gpurun_out/bench_$n.log | cut -c1-160)"
  done
fi
