for v in ST2 ST3 ST2 ST3; do for a in "pipeline 2"; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py $a 2>&1 | tail -1 | sed "s/^/$v /"; done; done > gpurun_out/st3_time.log 2>&1
PARADL_LIB=$PWD/exp/libST3.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "pipeline or full_sweep or sharded or config" > gpurun_out/gpu_st3.log 2>&1; echo "tests rc=$?"
