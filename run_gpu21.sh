export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_mr.log 2>&1; echo "tests rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_launches2.csv python tools/prof_pipeline.py pipeline 2 > gpurun_out/warm2.log 2>&1; echo "ncu rc=$?"
for v in MV2 MR MV2 MR; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py pipeline 2 2>&1 | tail -1 | sed "s/^/$v /"; done > gpurun_out/mr_time.log 2>&1
