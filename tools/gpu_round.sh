set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r1_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r1_pytest.log
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/r1_bench.out 2> gpurun_out/r1_bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/r1_bench.out
timeout 900 python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/r1_ref.out 2> gpurun_out/r1_ref.err; echo ref rc=$?
tail -c 2000 gpurun_out/r1_ref.out
