timeout 600 python -m tests.parity_report onestep frames30:2 2 2>&1 | tail -9
timeout 600 python -m tests.parity_report frame1 1 2 3 8 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q -s 2>&1 | grep -E "^E  .*assert|passed|failed|FAILED|frame1 n=" | head -20
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1000
