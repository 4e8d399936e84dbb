timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2as_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r2as_pytest.log
for r in 1 2; do
timeout 600 python bench.py --shape deepseek --extra-configs "" --no-cpu-baseline --steps 8 > gpurun_out/r2as_ds_$r.out 2>/dev/null
python tools/bench_summary.py gpurun_out/r2as_ds_$r.out 2>/dev/null | sed -n '1p;3p' | cut -c1-240
done
