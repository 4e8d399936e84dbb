"""Print the PCIe calibration samples (the transfer fit's inputs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200.calibration import measure_samples  # noqa: E402

for x in measure_samples(4096, 14336, gpu_loads=(1, 256), cpu_loads=(1,)):
    if x.device == "pcie":
        print(f"{x.load / 1e6:.1f} MB {x.duration * 1e3:.3f} ms {x.load / x.duration / 1e9:.1f} GB/s")
