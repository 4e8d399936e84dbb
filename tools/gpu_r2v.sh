# host decode prologue-prefetch A/B (B200 box host), interleaved
for r in 1 2; do
for v in 1 0; do echo "== HM_PF_PROLOGUE=$v"; HM_PF_PROLOGUE=$v NT=16 timeout 300 python tools/host_phase_prof.py; done
done
