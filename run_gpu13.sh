export PATH=/usr/local/cuda/bin:$PATH
for e in 1 0 1 0; do for a in "pipeline 2" "all 2"; do PARADL_NO_STRUCT_TABLE=$e timeout 120 python tools/prof_pipeline.py $a 2>&1 | tail -1 | sed "s/^/off=$e /"; done; done > gpurun_out/st_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_st.log 2>&1; echo "tests rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_st python tools/prof_pipeline.py pipeline 2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/st_launches.csv python tools/prof_pipeline.py all 2 > /dev/null 2>&1; echo "ncu2 rc=$?"
