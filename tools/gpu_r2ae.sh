# 4-bit GEMV chunk sweep (Mixtral / DeepSeek / Qwen2, 1-8 experts)
for c1 in 8 16 32; do for c2 in 0 16 48; do echo "== HM_Q4_CHUNK1=$c1 HM_Q4_CHUNK2=$c2"; HM_Q4_CHUNK1=$c1 HM_Q4_CHUNK2=$c2 timeout 300 python tools/q4_bench.py 1,2,8 2>&1 | grep -E "^(mixtral|deepseek|qwen2)" | tr '\n' ' '; echo; done; done
