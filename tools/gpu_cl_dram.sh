# DRAM bytes of k_pcg_cl per launch (ncu, a subset of metrics) on the config-5 PDE alone
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/d_build.log 2>&1
timeout 300 python tools/pde_bench.py --config 5 --nb 4736 --reps 1 > gpurun_out/d_plain.log 2>&1 && timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_pcg_cl -s 1 -c 1 python tools/pde_bench.py --config 5 --nb 4736 --reps 1 > gpurun_out/d_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "dram__|gpu__time" gpurun_out/d_ncu.log; tail -1 gpurun_out/d_plain.log
