"""Run tools/fp64_peak (burst + 3 s sustained per kernel) with nvidia-smi
clocks sampled during the run; write profiles/<out>.json with the peaks and
the clock record (median SM MHz under load, max, throttle reasons).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
    python tools/fp64_peak_clocks.py profiles/r02_fp64_peak.json
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (ClockSampler)

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
exe = os.path.join(ROOT, "tools", "fp64_peak")
clk = bench.ClockSampler(0)
clk.start()
res = subprocess.run([exe, "3"], capture_output=True, text=True, check=True)
c = clk.stop()
d = json.loads(res.stdout.strip().splitlines()[-1])
d["clocks"] = c
d["how"] = ("tools/fp64_peak.cu: 8 CTAs/SM x 256 threads; DFMA 8 independent chains; DMMA m16n8k4 / m16n8k16 "
            "4 / 2 independent accumulators; burst = one launch after a warm-up, sustained = back to back for 3 s "
            "per kernel; CUDA events; 2 flops per FMA")
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
