# host decode prefetch distance / clamp sweep, DeepSeek n=1..4 and Mixtral n=1
export NT=16 HM_PF_PROLOGUE=0
for v in "HM_PF_DIST=32768" "HM_PF_DIST=4096" "HM_PF_DIST=8192" "HM_PF_DIST=12288" "HM_PF_CLAMP=1" "HM_PF_CLAMP=1 HM_PF_DIST=16384" "HM_PF_CLAMP=1 HM_PF_DIST=8192" "HM_PF_DIST=8192 HM_DECODE_GRAIN=0" "HM_PF_DIST=32768"; do
echo "== $v"; env $v timeout 300 python tools/host_phase_prof.py
done
