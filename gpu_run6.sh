for k in k_render k_onesweep k_emit k_preprocess; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 6 -c 2 -o gpurun_out/prof_${k} python bench.py --ncu --steps 1 --warmup 1 --views-per-step 2 > /dev/null 2>&1; echo $k=$?
done
