# K6b table / block-shape variants (scripts/build_variants.sh builds them): ms per frames30 step,
# K5 and K6 ms per iteration
mkdir -p gpurun_out
# (variants were built with -DMRF_BLK_LOG / MRF_BLK_CTAS / MRF_BLK_ROWS, macros since removed)
for v in base t12c4 t12c4r32 t11r8 t12c5 base; do
  if [ $v = base ]; then L=""; else L="MRF_LIB=paper_2006_03512_b200/variants/libmrf_$v.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/v_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["roofline"]["ms_k5"],3), round(d["roofline"]["ms_k6"],3), d["roofline"]["k6_path"], d["clocks"]["reasons"])' 2>&1 | tail -1)"
done
