for v in D0 D1; do for a in "pipeline 2" "all 2" "pd 5" "pipeline 3"; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py $a 2>&1 | tail -1 | sed "s/^/$v /"; done; done > gpurun_out/d_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests9.log 2>&1; echo "tests rc=$?"
