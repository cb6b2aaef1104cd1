"""Time k_pcg_cl builds with different per-mesh register choices (pcg_cl.cuh: USFFT_CL_PSM / _DG /
_TZ as functions of n): python tools/cl_variants.py "TZ=0" "TZ=(nn)==64" ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_04131_b200 import build

for k, spec in enumerate(sys.argv[1:]):
    out = f"/tmp/libusfft_v{k}.so"
    defs = [f"-DUSFFT_CL_{kv.split('=')[0]}(nn)=({kv.split('=', 1)[1]})" for kv in spec.split(",")]
    subprocess.run([build.NVCC, *build.FLAGS, *defs, "-o", out, *build.sources()], cwd=build.SRC, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    for cfg in (5, 3):
        code = (f"import sys; sys.path.insert(0, {ROOT!r}); from paper_2109_04131_b200 import _native; _native.LIB_PATH={out!r}; "
                f"sys.argv=['x','--config','{cfg}','--nb','70000']; import runpy; runpy.run_path({ROOT + '/tools/pde_bench.py'!r}, run_name='__main__')")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(spec, "config", cfg, "ms %.2f" % d["ms"], "iters", d["iters_mean"], flush=True)
        except Exception:
            print(spec, "config", cfg, "FAILED", r.stderr[-300:], flush=True)
