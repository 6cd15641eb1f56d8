mkdir -p gpurun_out
V=paper_2006_03512_b200/variants
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/k_variants.py --repeat 2 "" > gpurun_out/var_base.log 2>&1
MRF_LIB=$V/libmrf_w8.so python scripts/k_variants.py --repeat 2 "" > gpurun_out/var_w8.log 2>&1
MRF_LIB=$V/libmrf_w32.so python scripts/k_variants.py --repeat 2 "" > gpurun_out/var_w32.log 2>&1
cat gpurun_out/var_base.log gpurun_out/var_w8.log gpurun_out/var_w32.log
