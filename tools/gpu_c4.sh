# config-4 round: launch list (which kernels the streamed selection spends its time in)
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/c4_build.log 2>&1
timeout 900 python bench.py --config 4 --t 3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c4_plain.json 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/c4_launches.csv python bench.py --config 4 --t 3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c4_ncu.log 2>&1; echo "rc=$?"
