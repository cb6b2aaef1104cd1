# k_pcg_cl v3 check on one B200: PDE parity tests for n = 64, 128, PDE-only timing, phase probe.
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/c3_build.log 2>&1; echo "build rc=$?"
timeout 300 python tools/pde_bench.py --config 5 --nb 4736 --reps 3 > gpurun_out/c3_pde5.txt 2>&1; echo "pde5 rc=$?"; cat gpurun_out/c3_pde5.txt | tail -3
timeout 300 python tools/pde_bench.py --config 3 --nb 8192 --reps 3 > gpurun_out/c3_pde3.txt 2>&1; echo "pde3 rc=$?"; cat gpurun_out/c3_pde3.txt | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sample_pde or pcg" > gpurun_out/c3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c3_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_checkpoint.py -x -q -k "whole_round or resume or refused" > gpurun_out/c3_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/c3_full.log
timeout 300 python tools/cl_probe.py --config 5 > gpurun_out/c3_probe5.txt 2>&1; echo "probe5 rc=$?"; grep -v warning gpurun_out/c3_probe5.txt | tail -20
