"""Per-kernel device times of one call (torch.profiler / CUPTI): python scripts/kprof.py <script> [args...]
Runs the target script's module-level code once for warm-up inside the profiler, then prints
a per-kernel summary of everything launched."""
import os, runpy, sys
from torch.profiler import ProfilerActivity, profile
sys.argv = sys.argv[1:]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    runpy.run_path(sys.argv[0], run_name="__main__")
rows = sorted(prof.key_averages(), key=lambda e: -getattr(e, "self_device_time_total", 0))
for e in rows[:25]:
    t = getattr(e, "self_device_time_total", 0)
    if t > 0:
        print(f"{t/1e3:9.3f} ms total  n={e.count:5d}  avg {t/max(e.count,1):8.1f} us  {e.key[:100]}")
