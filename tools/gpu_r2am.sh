# host decode steal-unit sweep (isolated), interleaved
for r in 1 2 3; do for kb in 16 32 64; do echo "== HM_STEAL_KB=$kb"; for sh in deepseek:1,2,3 qwen2:1,3 mixtral:1; do HM_STEAL_KB=$kb ONLY=$sh NT=16 timeout 300 python tools/host_phase_prof.py | sed 's/start max.*phase2/phase2/'; done; done; done
