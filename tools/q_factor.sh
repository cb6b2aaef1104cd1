for c in periodic_mu1.2 affine_example lognormal_example; do for f in 1 4 16; do timeout 900 python tools/full_run.py --config $c --n-test 10000 --lattice-factor $f 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['workload'], 'f=%d' % d['lattice_factor'], 'q=%.2f' % d['q'], 'samples=%d' % (d['samples_detection']+d['samples_step3']), 'err2max=%.2e' % d['err2_max'], 'ms=%.0f' % d['ms_detection'])
" ; done; done
