# Bounds-checked build (-DUSFFT_BOUNDS: device asserts on every computed shared-memory / DSMEM
# index of k_pcg_cl and k_fft_rader_r) run over small and full-size cases on one B200:
#   bash tools/bounds_check.sh     (compute-sanitizer is closed on this pool)
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/bc_build.log 2>&1
import subprocess, sys
sys.path.insert(0, ".")
from paper_2109_04131_b200 import build
cmd = [build.NVCC, *build.FLAGS, "-DUSFFT_BOUNDS", "-o", "/tmp/libusfft_bounds.so", *build.sources()]
r = subprocess.run(cmd, cwd=build.SRC)
sys.exit(r.returncode)
PY
echo "bounds build rc=$?"
USFFT_LIB=/tmp/libusfft_bounds.so timeout 900 python tools/sanitize_run.py > gpurun_out/bc_small.log 2>&1; echo "small rc=$?"; tail -3 gpurun_out/bc_small.log
USFFT_LIB=/tmp/libusfft_bounds.so timeout 900 python tools/pde_bench.py --config 5 --nb 1184 --reps 1 > gpurun_out/bc_pde5.log 2>&1; echo "pde5 rc=$?"; tail -1 gpurun_out/bc_pde5.log
USFFT_LIB=/tmp/libusfft_bounds.so timeout 900 python tools/pde_bench.py --config 3 --nb 2048 --reps 1 > gpurun_out/bc_pde3.log 2>&1; echo "pde3 rc=$?"; tail -1 gpurun_out/bc_pde3.log
USFFT_LIB=/tmp/libusfft_bounds.so timeout 900 python tools/fft_bench.py > gpurun_out/bc_fft.log 2>&1; echo "fft rc=$?"; tail -3 gpurun_out/bc_fft.log
USFFT_LIB=/tmp/libusfft_bounds.so timeout 900 python -m pytest tests/test_gpu_keys_product.py -q > gpurun_out/bc_keys.log 2>&1; echo "keys rc=$?"; tail -1 gpurun_out/bc_keys.log
