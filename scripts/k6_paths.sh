mkdir -p gpurun_out
for em in 1 2 4 8; do for k6 in block tile; do
  MRF_K6=$k6 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 --emulate-ranks $em > gpurun_out/e_${k6}_${em}.log 2>&1
  echo "frames30 em=$em k6=$k6 $(tail -1 gpurun_out/e_${k6}_${em}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["kernel_ms_per_step"].get("voxel_sum"), d["kernel_ms_per_step"].get("dda_fill"), d["kernel_ms_per_step"].get("transpose"))' 2>&1 | tail -1)"
done; done
for k6 in tile block; do
  MRF_K6=$k6 timeout 600 python bench.py --config frames100 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/f100_${k6}.log 2>&1
  echo "frames100 k6=$k6 $(tail -1 gpurun_out/f100_${k6}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["kernel_ms_per_step"].get("voxel_sum"), d["kernel_ms_per_step"].get("dda_fill"), d["kernel_ms_per_step"].get("transpose"))' 2>&1 | tail -1)"
done
