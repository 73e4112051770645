export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_lw.log 2>&1; echo "tests rc=$?"
for a in data_lw gpipe spatial_ag; do timeout 120 python tools/prof_next.py $a; done > gpurun_out/lw_time.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_lw python tools/prof_next.py data_lw > /dev/null 2>&1; echo "ncu rc=$?"
