# host worker thread pinning A/B in the Mixtral bench (no children, no CPU baseline), interleaved
for r in 1 2; do for v in 0 1; do
HM_PIN_THREADS=$v timeout 600 python bench.py --extra-configs "" --no-cpu-baseline > gpurun_out/r2ag_pin${v}_$r.out 2>/dev/null
python tools/bench_summary.py gpurun_out/r2ag_pin${v}_$r.out | head -3 | sed "s/^/pin=$v run=$r /" | cut -c1-250
done; done
