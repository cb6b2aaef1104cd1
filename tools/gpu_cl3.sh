mkdir -p gpurun_out
bash tools/gpu_cl2.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_cl -c 1 -o gpurun_out/cl5v2 -f python tools/pde_bench.py --config 5 --nb 2368 --reps 1 > gpurun_out/ncu_cl5v2.log 2>&1; tail -1 gpurun_out/ncu_cl5v2.log
