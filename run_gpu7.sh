export PATH=/usr/local/cuda/bin:$PATH
for v in G1 T1; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_next.py gpipe 2>&1 | tail -1 | sed "s/^/$v /"; done > gpurun_out/gp_time7.log 2>&1
timeout 120 python tools/prof_next.py spatial_ag >> gpurun_out/gp_time7.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "next or gpipe or random_corpus or explain" > gpurun_out/gpu_next7.log 2>&1; echo "tests rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_gpipe3 python tools/prof_next.py gpipe > gpurun_out/ncu_gpipe3.log 2>&1; echo "ncu rc=$?"
