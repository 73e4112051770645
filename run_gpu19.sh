export PATH=/usr/local/cuda/bin:$PATH
for v in MV MV2 MV MV2; do for a in "pipeline 2" "all 2"; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py $a 2>&1 | tail -1 | sed "s/^/$v /"; done; done > gpurun_out/mv2_time.log 2>&1
PARADL_LIB=$PWD/exp/libMV2.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_mv2.log 2>&1; echo "tests rc=$?"
PARADL_LIB=$PWD/exp/libMV2.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv2_launches.csv python tools/prof_pipeline.py all 2 > /dev/null 2>&1; echo "ncu2 rc=$?"
