timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|assert|^E |passed|failed" | head -20
timeout 600 python -m tests.parity_report onestep frames30:2 2 2>&1 | tail -9
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1200
python -c "from paper_2006_03512_b200 import _build; _build.build(force=True, extra=['-DMRF_LANE_K=16','-DMRF_K5_MIN_BLOCKS=2'])"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench16.log 2>&1; tail -1 gpurun_out/bench16.log | cut -c1-1200
