for r in 1 2; do for v in K0 K1 K2 K3; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_pipeline.py pipeline 2 2>&1 | tail -1 | sed "s/^/$v /"; done; done > gpurun_out/k_time.log 2>&1
