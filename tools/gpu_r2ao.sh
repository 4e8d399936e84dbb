# steal size A/B in the Mixtral bench on one box, interleaved
for r in 1 2 3; do for kb in 64 256; do
HM_STEAL_KB=$kb timeout 600 python bench.py --extra-configs "" --no-cpu-baseline > gpurun_out/r2ao_${kb}_$r.out 2>/dev/null
python - <<PY
import json
d=json.loads([x for x in open("gpurun_out/r2ao_${kb}_$r.out") if x.startswith("{")][-1])
print("steal=$kb run=$r value %.2f e2e %.2f worker %.0f probe %.0f" % (d["value"], d["e2e"]["value"], d["step_roofline"]["host_worker_gbs"], d["step_roofline"]["host_read_probe_gbs"]))
PY
done; done
