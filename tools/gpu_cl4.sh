mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/c4_build.log 2>&1; echo "build rc=$?"
timeout 300 python tools/cl_probe.py --config 5 > gpurun_out/c4_probe5.txt 2>&1; echo "probe5 rc=$?"; grep -v warning gpurun_out/c4_probe5.txt | tail -20
timeout 300 python tools/pde_bench.py --config 5 --nb 1184 --reps 1 > gpurun_out/c4_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_cl -c 1 -o gpurun_out/c4_cl5 -f python tools/pde_bench.py --config 5 --nb 1184 --reps 1 > gpurun_out/c4_ncu5.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/c4_ncu5.log
