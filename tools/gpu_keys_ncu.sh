mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/kn_build.log 2>&1
timeout 900 python bench.py --config 4 --t 3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/kn_plain.json 2>&1 && timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_kappa_tiled|k_select" -c 2 -o gpurun_out/kn_full -f python bench.py --config 4 --t 3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/kn_ncu.log 2>&1; echo "rc=$?"
