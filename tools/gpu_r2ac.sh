# AMX expert: algo 0 (per-unit full-K) vs algo 1 (cache-blocked), three shapes
for a in 0 1; do for sh in "2048 1408" "4096 14336" "3584 2560"; do echo "== algo $a $sh"; HM_AMX_ALGO=$a timeout 300 python tools/amx_phase_prof.py $sh | cut -c1-40; done; done
