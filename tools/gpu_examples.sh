set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py > gpurun_out/bench_ex.json 2>gpurun_out/bench_ex.err; tail -1 gpurun_out/bench_ex.json | cut -c1-600
for c in lognormal_example affine_example; do timeout 900 python tools/full_run.py --config $c --n-test 10000 2>&1 | tail -1; done
