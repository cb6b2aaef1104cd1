for c in periodic_mu1.2 periodic_mu3.6 affine_example; do timeout 900 python tools/fixed_sets.py --config $c --N 4 8 16 32 --n-test 10000 2>&1 | grep "^{" ; done
