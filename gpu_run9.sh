timeout 300 python profiles/host_overhead.py > gpurun_out/host_overhead.txt 2>&1; head -30 gpurun_out/host_overhead.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-score > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['stages_ms'], d['host_enqueue_ms_per_frame'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > /dev/null 2>&1; echo ncu1=$?
