"""Summarise an ncu CSV capture of one synthesis + analysis per width
(tools/prof_run.py) into per-phase DRAM traffic per launch.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_run.py c2
    python tools/ncu_traffic.py gpurun_out/traffic.csv c2 profiles/r01_traffic_c2.json

Phases are told apart by kernel name: fwd_kernel -> fwd@1, adj_kernel -> adj@1,
mma_kernel<S, false, ...> -> fwd@W, mma_kernel<S, true, ...> -> adj@W (W = the
workload's multi-RHS width), reduce_kernel -> the adjoint group sums.  bench.py
reads the output as the roofline's ``traffic`` (bytes per launch, averaged over
the phase's launches in one apply, the same averaging as ``achieved``).
"""
from __future__ import annotations

import csv
import json
import sys
from collections import defaultdict

UNITS = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def phase_of(name: str, width: int) -> str | None:
    if name.startswith("void") or "::" in name:
        name = name.split("::")[-1]
    if name.startswith("fwd_kernel") or name.startswith("fwd_lat_kernel"):
        return "fwd@1"
    if name.startswith("adj_kernel"):
        return "adj@1"
    if name.startswith("mma_kernel") or name.startswith("mma_ws_kernel") or name.startswith("mma_real_kernel"):
        args = name[name.index("<") + 1:].split(",")
        # mma_real_kernel<ADJ, ...>, mma_ws_kernel<ADJ>, mma_kernel<S, ADJ, ...>
        flag = args[1] if name.startswith("mma_kernel") else args[0]
        adj = flag.strip().rstrip(">") in ("1", "true")
        return f"{'adj' if adj else 'fwd'}@{width}"
    if name.startswith("reduce_kernel"):
        return "sum"
    return None


def main(src: str, workload: str, dst: str, width: int = 32):
    rows = list(csv.reader(l for l in open(src) if not l.startswith("==")))
    head = rows[0]
    col = {h: i for i, h in enumerate(head)}
    per = defaultdict(lambda: defaultdict(float))
    units = {}
    for r in rows[1:]:
        if len(r) < len(head):
            continue
        metric, unit, val = r[col["Metric Name"]], r[col["Metric Unit"]], r[col["Metric Value"]]
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        v *= UNITS.get(unit.lower(), 1.0)
        key = (r[col["ID"]], r[col["Kernel Name"]])
        per[key][metric] = v
        units[metric] = unit
    out = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
    for (_, name), ms in per.items():
        ph = phase_of(name, width)
        if ph is None:
            continue
        o = out[ph]
        o["launches"] += 1
        o["dram_bytes"] += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
        o["ms"] += ms.get("gpu__time_duration.sum", 0.0)
    res = {"workload": workload, "source": src.split("/")[-1],
           "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      f"--clock-control none python tools/prof_run.py {workload}",
           "phases": {}}
    for ph, o in sorted(out.items()):
        res["phases"][ph] = {"launches": o["launches"], "dram_bytes_total": o["dram_bytes"],
                             "dram_bytes_per_launch": o["dram_bytes"] / max(o["launches"], 1),
                             "ms_total_cold_serialised": o["ms"]}
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 4:
        wd = int(sys.argv[4])
    else:  # the workload's multi-RHS width (tools/prof_run.py runs nrhs = 1 and that width)
        import os
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import mht_inputs as mi
        wd = max([r for r in mi.WORKLOADS[sys.argv[2]].nrhs if r > 1] or [32])
    main(sys.argv[1], sys.argv[2], sys.argv[3], wd)
