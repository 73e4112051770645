timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests44.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench44.log 2>&1; echo "bench rc=$?"
