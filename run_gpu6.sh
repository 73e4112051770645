export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests6.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke6.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench6.log 2>&1; echo "bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_gpipe2 python tools/prof_next.py gpipe > gpurun_out/ncu_gpipe2.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 3 -f -o gpurun_out/full_spag python tools/prof_next.py spatial_ag > gpurun_out/ncu_spag.log 2>&1; echo "ncu2 rc=$?"
