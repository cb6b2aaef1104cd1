# State check on one B200: build, GPU tests, default bench line (config 5), reference arm,
# config-2 line, ncu launch list of the default bench.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/st_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/st_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/st_tests.log
timeout 600 python bench.py > gpurun_out/st_bench.json 2> gpurun_out/st_bench.err; echo "bench rc=$?"; cat gpurun_out/st_bench.json
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/st_bench_c2.json 2> gpurun_out/st_bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/st_ref.json 2> gpurun_out/st_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/st_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/st_ncu.log 2>&1; echo "ncu rc=$?"
