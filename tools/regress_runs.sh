for c in 1 2 periodic_mu1.2 affine_example; do timeout 600 python tools/full_run.py --config $c --n-test 10000 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['workload'], 'nI', d['nI'], 'samples', d['samples_detection'] + d['samples_step3'], 'err2max %.3e' % d['err2_max'], 'ms det %.0f s3 %.0f err %.0f' % (d['ms_detection'], d['ms_step3'], d['ms_errors']))"; done
timeout 600 python tools/full_run.py --config lognormal_example --lattice-factor 4 --n-test 10000 2>&1 | tail -1 | cut -c1-300
