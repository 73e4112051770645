timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "next or gpipe or random_corpus or explain" > gpurun_out/gpu_next2.log 2>&1; echo "tests rc=$?"
for v in G0 G1; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_next.py gpipe 2>&1 | tail -1 | sed "s/^/$v /"; done > gpurun_out/gp_time.log 2>&1
PARADL_LIB=$PWD/exp/libG1.so timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "next or gpipe or random_corpus" > gpurun_out/gpu_next3.log 2>&1; echo "tests G1 rc=$?"
