timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['stages_ms'], d['host_enqueue_ms_per_frame'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_render$' -s 2 -c 1 -o gpurun_out/prof_k_render python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > /dev/null 2>&1; echo ncu2=$?
