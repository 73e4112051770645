export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_sk.log 2>&1; echo "tests rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_launches4.csv python tools/prof_pipeline.py pipeline 2 > gpurun_out/warm4.log 2>&1; echo "ncu rc=$?"
for v in MS SK MS SK; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py pipeline 2 2>&1 | tail -1 | sed "s/^/$v /"; done > gpurun_out/sk_time.log 2>&1
