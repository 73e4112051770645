timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "struct_mode or full_sweep_topk or sharded" > gpurun_out/gpu_s4.log 2>&1; echo "s4 tests rc=$?"
for e in 1 0 1 0; do PARADL_NO_STRUCT_MODE=$e timeout 120 python tools/prof_pipeline.py pipeline 2 2>&1 | tail -1 | sed "s/^/off=$e /"; done > gpurun_out/s4_time.log 2>&1
PARADL_NO_STRUCT_MODE=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_s4 python tools/prof_pipeline.py pipeline 2 > /dev/null 2>&1; echo "ncu rc=$?"
