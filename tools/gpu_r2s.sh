# re-entry check: smoke, all gpu tests, default bench (own arm + reference arm), launch list
TAG=${TAG:-r2s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E 'Model name|Socket|NUMA node\(s\)|^CPU\(s\)'
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/${TAG}_pytest.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.out 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
tail -c 6000 gpurun_out/${TAG}_bench.out
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.out 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
tail -c 2000 gpurun_out/${TAG}_ref.out
