for r in 1 2; do for v in 1 0; do for sh in "2048 1408" "4096 14336"; do echo "== pf $v $sh"; HM_AMX_UNIT_PF=$v timeout 300 python tools/amx_phase_prof.py $sh | cut -c1-40; done; done; done
