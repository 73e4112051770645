set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/bench_c5.log 2>&1; echo "bench5 rc=$?"
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/bench_c3.log 2>&1; echo "bench3 rc=$?"
tail -3 gpurun_out/*.log
