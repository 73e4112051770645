export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1; echo "launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_c2_pipeline python tools/prof_pipeline.py pipeline 2 > gpurun_out/ncu_full_c2.log 2>&1; echo "full c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_c5_pd python tools/prof_pipeline.py pd 5 > gpurun_out/ncu_full_c5.log 2>&1; echo "full c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full_c3_pipeline python tools/prof_pipeline.py pipeline 3 > gpurun_out/ncu_full_c3.log 2>&1; echo "full c3 rc=$?"
