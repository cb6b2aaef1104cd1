# Round refresh on one B200: GPU tests + smoke, default bench (config 5), configs 2-4, reference
# arm, launch list of the default bench, ncu --set full of k_pcg_cl and k_fft_rader_r inside the
# timed region (cudaProfilerStart/Stop).  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/r_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r_smoke.log
timeout 600 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?"; cat gpurun_out/r_bench.json
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r_bench_c2.json 2> gpurun_out/r_bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r_bench_c3.json 2> gpurun_out/r_bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config 4 --t 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r_bench_c4.json 2> gpurun_out/r_bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r_ref.json 2> gpurun_out/r_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu.log 2>&1; echo "ncu-list rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r_plain1.json 2>&1 && timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_pcg_cl|k_fft_rader_r" -c 2 -o gpurun_out/r_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncufull.log 2>&1; echo "ncu-full rc=$?"
