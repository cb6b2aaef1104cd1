mkdir -p gpurun_out
python -m paper_2109_04131_b200.build > gpurun_out/f_build.log 2>&1
timeout 300 python tools/fft_bench.py > gpurun_out/fn_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fft_rader_r -s 12 -c 1 -o gpurun_out/fn_4001 -f python tools/fft_bench.py > gpurun_out/fn_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/fn_ncu.log
