# overlap of the layer's GPU launches with the host worker start: GPU tests + DeepSeek / Mixtral benches
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2ah_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2ah_pytest.log
for r in 1 2; do
timeout 600 python bench.py --shape deepseek --extra-configs "" --no-cpu-baseline --steps 8 > gpurun_out/r2ah_ds_$r.out 2>/dev/null
python tools/bench_summary.py gpurun_out/r2ah_ds_$r.out 2>/dev/null | head -3 | cut -c1-260
done
timeout 600 python bench.py --extra-configs "" --no-cpu-baseline > gpurun_out/r2ah_mx.out 2>/dev/null
python tools/bench_summary.py gpurun_out/r2ah_mx.out 2>/dev/null | head -3 | cut -c1-260
