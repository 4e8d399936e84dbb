for v in 2 1; do
HM_GEMV_FUSED=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ffn --csv python tools/gemv_lib_bench.py 3 deepseek,mixtral 1,4,6 > gpurun_out/r2f_ncu_v$v.csv 2>&1; echo ncu rc=$?
done
