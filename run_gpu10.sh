timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "struct_mode or full_sweep_topk or sharded" > gpurun_out/gpu_s3.log 2>&1; echo "s3 tests rc=$?"
for e in 1 0; do PARADL_NO_STRUCT_MODE=$e timeout 120 python tools/prof_pipeline.py pipeline 2 2>&1 | tail -1 | sed "s/^/off=$e /"; done > gpurun_out/s3_time.log 2>&1
PARADL_NO_STRUCT_MODE=0 timeout 120 python tools/prof_pipeline.py all 2 >> gpurun_out/s3_time.log 2>&1
