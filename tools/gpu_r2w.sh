# host decode knob sweep on the B200 box host, DeepSeek n=1,2
export ONLY=deepseek:1,2 NT=16 HM_PF_PROLOGUE=0
for v in "X=0" "HM_DECODE_GRAIN=0" "HM_DECODE_GRAIN=8" "HM_DECODE_GRAIN=32" "HM_DECODE_GRAIN=64" "HM_PF_DIST=8192" "HM_PF_DIST=16384" "HM_PF_DIST=65536" "HM_PF_HINT=0" "HM_PF_HINT=1" "HM_PF_HINT=3" "HM_DECODE_STEAL=0" "X=1"; do
echo "== $v"; env $v timeout 300 python tools/host_phase_prof.py
done
