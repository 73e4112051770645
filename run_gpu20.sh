export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_launches.csv python tools/prof_pipeline.py pipeline 2 > gpurun_out/warm.log 2>&1; echo "ncu rc=$?"
