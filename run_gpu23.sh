export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --set full --clock-control none --import-source on -k regex:struct_table -c 1 -f -o gpurun_out/full_stk python tools/prof_pipeline.py pipeline 2 > /dev/null 2>&1; echo "ncu rc=$?"
