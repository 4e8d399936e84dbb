# one GPU round: smoke, gpu tests, bench (own arm + reference arm); outputs under gpurun_out/$TAG_*
TAG=${TAG:-r2}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/${TAG}_bench.out 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
tail -c 4000 gpurun_out/${TAG}_bench.out
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.out 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
tail -c 2000 gpurun_out/${TAG}_ref.out
