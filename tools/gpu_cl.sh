set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 240 python tools/cl_check.py --config 3 --check 4 > gpurun_out/cl3.log 2>&1; echo "rc=$?" >> gpurun_out/cl3.log
tail -3 gpurun_out/cl3.log
timeout 300 python tools/cl_check.py --config 5 --check 3 > gpurun_out/cl5.log 2>&1; echo "rc=$?" >> gpurun_out/cl5.log
tail -3 gpurun_out/cl5.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pcg or fft_paths or keys or eval" > gpurun_out/t1.log 2>&1; tail -5 gpurun_out/t1.log
