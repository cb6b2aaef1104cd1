# one GPU session: tests, bench (config 5 default + config 2), launch list of the bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log; tail -3 gpurun_out/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.log 2> gpurun_out/bench5.err; echo "bench5 rc=$?"; tail -1 gpurun_out/bench5.log | head -c 3000; echo
timeout 300 python bench.py --steps 10 --warmup 3 --config 2 --no-cpu-baseline > gpurun_out/bench2.log 2> gpurun_out/bench2.err; echo "bench2 rc=$?"; tail -1 gpurun_out/bench2.log | head -c 1500; echo
timeout 60 python bench.py --gpus 2 --steps 1 --warmup 3 > gpurun_out/gpus2.log 2>&1; echo "gpus2 rc=$?"; tail -2 gpurun_out/gpus2.log
