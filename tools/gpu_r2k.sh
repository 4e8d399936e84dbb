start=$(date +%s)
timeout 1200 python bench.py --steps 8 --warmup 3 > gpurun_out/r2k_bench.out 2> gpurun_out/r2k_bench.err; echo bench rc=$?
echo elapsed $(( $(date +%s) - start ))
