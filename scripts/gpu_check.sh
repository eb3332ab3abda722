#!/bin/bash
# One gpurun call: build, GPU tests, default bench line, launch list, ncu full captures.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh TAG [tests|bench|launches|full]...'
TAG=${1:-run}; shift
STEPS=${@:-tests bench launches full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail gpurun_out/${TAG}_build.log; exit 1; }
for s in $STEPS; do case $s in
tests)
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/${TAG}_pytest_gpu.log ;;
smoke)
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_exit=$?; tail -3 gpurun_out/${TAG}_smoke.log ;;
bench)
  timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_exit=$?; tail -3 gpurun_out/${TAG}_bench.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['value'], d['stages_ms'], d.get('kernels_us'), d['roofline'])" ;;
bench2)
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench2.json 2> gpurun_out/${TAG}_bench2.err; echo bench2_exit=$?; tail -3 gpurun_out/${TAG}_bench2.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench2.json')); print(d['n_gpus'], d['value'], d['config']['process_group'], d['prune_score'])" ;;
benchfast)
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-score > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_exit=$?; tail -3 gpurun_out/${TAG}_bench.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['value'], d['stages_ms'], d.get('kernels_us'))" ;;
launches)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --ncu --no-backward --steps 1 --warmup 1 --views-per-step 2 > /dev/null 2>&1; echo ncu_launches=$?
  python profiles/summarize.py launches gpurun_out/${TAG}_launches.csv ;;
chain)
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/${TAG}_chain python scripts/profile_frame.py ${PROF_ARGS} > gpurun_out/${TAG}_chain.log 2>&1; echo ncu_chain=$?
  ncu -i gpurun_out/${TAG}_chain.ncu-rep --page raw --csv > gpurun_out/${TAG}_chain_raw.csv 2>/dev/null
  python profiles/summarize.py full gpurun_out/${TAG}_chain.ncu-rep > gpurun_out/${TAG}_chain.txt; head -3 gpurun_out/${TAG}_chain.txt ;;
prof)
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_render}" -o gpurun_out/${TAG}_prof python scripts/profile_frame.py ${PROF_ARGS} > gpurun_out/${TAG}_prof.log 2>&1; echo ncu_prof=$?
  ncu -i gpurun_out/${TAG}_prof.ncu-rep --page raw --csv > gpurun_out/${TAG}_prof_raw.csv 2>/dev/null ;;
sanitize)
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/${TAG}_sanitize_$tool.txt 2>&1; echo sanitize_$tool=$?; tail -2 gpurun_out/${TAG}_sanitize_$tool.txt
  done ;;
full)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_(preprocess|emit|render|onesweep|tile_finalize|render_backward|preprocess_backward)' -s 40 -c 12 -o gpurun_out/${TAG}_full python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > gpurun_out/${TAG}_full.log 2>&1; echo ncu_full=$? ;;
esac; done
