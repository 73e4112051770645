for v in G F; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/dense_time.py | sed "s/^/$v /" >> gpurun_out/dense45.log 2>&1; done
