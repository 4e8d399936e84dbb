# 4-bit host decode prefetch distance sweep (B200 box host)
export NT=16 Q4=1
for v in 16384 2048 4096 8192 32768 0 16384; do
echo "== HM_Q4_PF=$v"; HM_Q4_PF=$v timeout 300 python tools/host_phase_prof.py | sed 's/start max.*|//'
done
