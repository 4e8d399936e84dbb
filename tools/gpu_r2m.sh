out=gpurun_out/prof_r02b; mkdir -p $out
# grouped GEMM at a compute-bound shape (1024 tokens per expert) -- tensor-pipe counter
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 2 -c 2 -o $out/expert_gemm_m1024 \
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2504_05897_b200.microbench import gemm_bench
print(gemm_bench(4096, 14336, rows_per_expert=1024, n_experts=4, reps=2))" > $out/gemm1024.log 2>&1; echo ncu1 rc=$?
# un-profiled timing of the same shapes
python -c "
import sys, json; sys.path.insert(0, '.')
from paper_2504_05897_b200.microbench import gemm_bench
for m in (256, 512, 1024, 2048):
    print(m, json.dumps(gemm_bench(4096, 14336, rows_per_expert=m, n_experts=4, reps=4)))" > $out/gemm_sweep.log 2>&1; echo sweep rc=$?
cat $out/gemm_sweep.log
# 4-bit GEMV, Mixtral 1 and 4 experts, full set
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffn[12]_q4" -s 6 -c 2 -o $out/q4_mixtral1 \
  python tools/q4_bench.py 1 > /dev/null 2>&1; echo ncu2 rc=$?
