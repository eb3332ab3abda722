set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_render$' -s 6 -c 1 -o gpurun_out/prof_render python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > gpurun_out/ncu_full_render.log 2>&1; echo ncu2=$?
ls -la gpurun_out
