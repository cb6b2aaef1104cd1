for c in "$@"; do echo "== config $c"; timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), {k:d['config'][k] for k in ('M','L','samples_per_step','nJ','cg_iters_mean')}, 'frac', round(d['roofline']['frac'],4), d['roofline']['kernel'][:10], 'e2e', round(d['e2e']['value']), d['phase_ms_per_step'])
" 2>&1 | tail -1; tail -1 gpurun_out/bench_c$c.err; done
