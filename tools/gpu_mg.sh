# k_pcg_mg check on one B200: PDE-only timing at configs 1-2, parity tests of the n <= 32 paths
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/m_build.log 2>&1; echo "build rc=$?"
for c in 2 1; do timeout 300 python tools/pde_bench.py --config $c --nb 6817 --reps 5 > gpurun_out/m_pde$c.txt 2>&1; echo "pde$c rc=$?"; tail -1 gpurun_out/m_pde$c.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_examples.py -x -q -k "sample_pde or pcg or config1 or whole_round or stage or examples or lockstep" > gpurun_out/m_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m_tests.log
