# lattice-FFT check on one B200: parity tests and config-shaped timing
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/f_build.log 2>&1; echo "build rc=$?"
timeout 300 python tools/fft_bench.py > gpurun_out/f_bench.txt 2>&1; echo "bench rc=$?"; cat gpurun_out/f_bench.txt | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -x -q -k "fft or lattice or stage or round" > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f_tests.log
