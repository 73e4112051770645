export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench17.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense --no-next > gpurun_out/bench17_c5.log 2>&1; echo "bench5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches17.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-next > gpurun_out/ncu17.log 2>&1; echo "launch rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/full17_c2 python tools/prof_pipeline.py pipeline 2 > /dev/null 2>&1; echo "ncu rc=$?"
