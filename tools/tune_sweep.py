"""Run the plan autotuner over shapes and report the winning plan per shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_00076_b200 import engine
sizes = [int(x) for x in sys.argv[1:]] or [512, 768, 1024, 1280, 1536, 1792, 2048, 2304, 2816, 3328]
for s in sizes:
    plan, ms = engine.tune(s, s, s, reps=5)
    print(f"{s}^3: plan {plan}  {ms*1e3:.1f} us  {2*s**3/ms/1e9:.1f} TF", flush=True)
for (m, n, k) in [(16384, 16384, 256), (4093, 4099, 2047)]:
    plan, ms = engine.tune(m, n, k, reps=3)
    print(f"{m}x{n}x{k}: plan {plan}  {ms:.3f} ms  {2*m*n*k/ms/1e9:.1f} TF", flush=True)
