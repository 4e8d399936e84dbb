timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --live-fixture gpurun_out/live_mixtral.json > gpurun_out/r2h_fixture.out 2> gpurun_out/r2h_fixture.err; echo fixture rc=$?
tail -c 600 gpurun_out/r2h_fixture.out
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/r2h_bench.out 2> gpurun_out/r2h_bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/r2h_bench.out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x -k "fused" > gpurun_out/r2h_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r2h_pytest.log
