# compute-sanitizer, ONE tool per gpurun call: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck
TOOL=${1:-memcheck}
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/san_build.log 2>&1
timeout 600 python tools/sanitize_run.py > gpurun_out/san_plain_$TOOL.log 2>&1; echo "plain rc=$?"
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$TOOL.log 2>&1; echo "$TOOL rc=$?"
tail -15 gpurun_out/san_$TOOL.log
