mkdir -p gpurun_out
C="python scripts/k_variants.py --repeat 1 --iters 2 MRF_K5=class"
timeout 600 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'ray_msg_kernel' -s 6 -c 4 -o gpurun_out/prof_class -f $C > gpurun_out/ncu_class.log 2>&1
tail -2 gpurun_out/ncu_class.log
