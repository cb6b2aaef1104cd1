mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_cl -c 1 -o gpurun_out/cl5 -f python tools/pde_bench.py --config 5 --nb 2368 --reps 1 > gpurun_out/ncu_cl5.log 2>&1
tail -3 gpurun_out/ncu_cl5.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_cl -c 1 -o gpurun_out/cl3 -f python tools/pde_bench.py --config 3 --nb 4736 --reps 1 > gpurun_out/ncu_cl3.log 2>&1
tail -3 gpurun_out/ncu_cl3.log
