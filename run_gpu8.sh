for v in T1 Q2 Q4; do PARADL_LIB=$PWD/exp/lib$v.so timeout 120 python tools/prof_next.py gpipe 2>&1 | tail -1 | sed "s/^/$v /"; done > gpurun_out/gp_time8.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 -k "next or gpipe or random_corpus" > gpurun_out/gpu_next8.log 2>&1; echo "tests rc=$?"
