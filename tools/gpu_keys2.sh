mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/k_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_keys_product.py tests/test_gpu_streamed.py tests/test_gpu_parity.py -k "keys or select or streamed or carry or round or union" -x -q > gpurun_out/k_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/k_tests.log
timeout 900 python bench.py --config 4 --t 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/k_c4.json 2> gpurun_out/k_c4.err; echo "c4 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/k_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['phase_ms_per_step'])"
