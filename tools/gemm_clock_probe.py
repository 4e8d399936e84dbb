"""SM clock and power while the grouped GEMM runs back to back (is the tensor
kernel power-capped?): nvidia-smi sampled every 20 ms in the background."""
import subprocess
import sys
import time

sys.path.insert(0, "/root/repo")
from paper_2504_05897_b200.microbench import gemm_bench  # noqa: E402

p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader", "-lms", "20"], stdout=subprocess.PIPE, text=True)
time.sleep(1.0)
t0 = time.time()
r = gemm_bench(4096, 14336, 256, 8, reps=3000)
dt = time.time() - t0
time.sleep(0.5)
p.terminate()
rows = [l for l in p.stdout.read().splitlines() if "MHz" in l]
print("gemm", round(r["ms"], 4), "ms/call", round(r["tflops"], 1), "TF/s over", round(dt, 2), "s")
for l in rows[::5]:
    print(l)
