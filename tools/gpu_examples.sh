set -x
timeout 900 python -m pytest tests/test_gpu_moments.py -x -q 2>&1 | tail -5
for c in 2 periodic_mu1.2 periodic_mu3.6 affine_example; do timeout 900 python tools/full_run.py --config $c --n-test 10000 2>&1 | tail -1; done
