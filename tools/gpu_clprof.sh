# k_pcg_cl evidence on one B200: phase probe (n = 128, 64), PDE-only timing, one ncu --set full capture.
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/cp_build.log 2>&1; echo "build rc=$?"
timeout 300 python tools/cl_probe.py --config 5 > gpurun_out/cp_probe5.txt 2>&1; echo "probe5 rc=$?"; cat gpurun_out/cp_probe5.txt
timeout 300 python tools/cl_probe.py --config 3 > gpurun_out/cp_probe3.txt 2>&1; echo "probe3 rc=$?"
timeout 300 python tools/pde_bench.py --config 5 --nb 4736 --reps 3 > gpurun_out/cp_pde5.txt 2>&1; echo "pde5 rc=$?"; cat gpurun_out/cp_pde5.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_cl -c 1 -o gpurun_out/cp_cl5 -f python tools/pde_bench.py --config 5 --nb 1184 --reps 1 > gpurun_out/cp_ncu5.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/cp_ncu5.log
