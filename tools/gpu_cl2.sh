mkdir -p gpurun_out
timeout 60 python tools/cl_check.py --config 3 --check 4 > gpurun_out/cl3.log 2>&1; echo "rc=$?" >> gpurun_out/cl3.log; tail -2 gpurun_out/cl3.log
timeout 90 python tools/cl_check.py --config 5 --check 3 > gpurun_out/cl5.log 2>&1; echo "rc=$?" >> gpurun_out/cl5.log; tail -2 gpurun_out/cl5.log
timeout 200 python tools/cl_probe.py --config 5 2>/dev/null | tail -22
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pcg" 2>&1 | tail -3
