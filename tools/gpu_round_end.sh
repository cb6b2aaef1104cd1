# Round-end refresh on one B200: GPU tests, the default bench line (+ reference arm), the bench
# line of configs 3-5, and the ncu launch list of the default bench.  Outputs under gpurun_out/.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fin_tests.log
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
for c in 3 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c$c.json 2> gpurun_out/fin_c$c.err; echo "c$c rc=$?"; done
timeout 900 python bench.py --config 4 --t 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err; echo "c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err; echo "c2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_pcg_cl|k_fft_rader_r|k_kappa_grouped" -c 3 -o gpurun_out/fin_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 python tools/cl_probe.py --config 5 2>&1 | grep "^[a-zA-Z]" | grep -v "Remark\|detected" > gpurun_out/fin_probe5.txt; timeout 300 python tools/cl_probe.py --config 3 2>&1 | grep "^[a-zA-Z]" | grep -v "Remark\|detected" > gpurun_out/fin_probe3.txt; echo "probes done"
timeout 300 python tools/fft_bench.py > gpurun_out/fin_fft_bench.txt 2>&1; echo "fft bench rc=$?"
