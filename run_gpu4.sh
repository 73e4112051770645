export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "next or gpipe" > gpurun_out/gpu_next.log 2>&1; echo "next tests rc=$?"
for a in gpipe spatial_ag; do timeout 120 python tools/prof_next.py $a; done > gpurun_out/next_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_next.log 2>&1; echo "bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_gpipe python tools/prof_next.py gpipe > gpurun_out/ncu_gpipe.log 2>&1; echo "ncu rc=$?"
