export PATH=/usr/local/cuda/bin:$PATH
for v in ST ST2 ST ST2; do for a in "pipeline 2" "all 2"; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py $a 2>&1 | tail -1 | sed "s/^/$v /"; done; done > gpurun_out/st2_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_st2.log 2>&1; echo "tests rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_st2 python tools/prof_pipeline.py pipeline 2 > /dev/null 2>&1; echo "ncu rc=$?"
