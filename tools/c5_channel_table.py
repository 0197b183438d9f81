#!/usr/bin/env python
"""Tabulate the per-vehicle service-channel share of the reference's DSRC simulator for the C5
sweep ("set each cloud's vm_throughput_kbps to the simulator's per-vehicle share at
density c under static1609 vs AAA").

Runs the UNMODIFIED reference (oracle/_ref/libvcsref.so: sim.cpp run_simulation + vc_throughput,
metrics.cpp:8-11 per_vehicle_throughput) with the reference benchmark's own settings (seed 42,
10,000 ms, tools/cli.cpp:19-20) for n = 1..128 vehicles and writes tests/golden/c5_channel.json.
The GPU box never runs this: bench_workloads.py reads the committed table.
"""
import ctypes as C
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    L = C.CDLL(str(ROOT / "oracle" / "_ref" / "libvcsref.so"))
    f = L.ref_per_vehicle_kbps
    f.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    table = {}
    for name, scheme in (("static1609", 0), ("aaa", 1)):
        row = []
        for n in range(1, 129):
            out = C.c_double()
            if f(n, scheme, 42, 10_000, C.byref(out)) != 0:
                raise RuntimeError(f"ref_per_vehicle_kbps({n}, {name}) failed")
            row.append(out.value)
        table[name] = row
    doc = {"source": "reference sim.cpp run_simulation + vc_throughput / n_vehicles "
                     "(metrics.cpp:8-11), seed 42, 10000 ms (tools/cli.cpp:19-20)",
           "n_vehicles": list(range(1, 129)), "per_vehicle_kbps": table}
    out = ROOT / "tests" / "golden" / "c5_channel.json"
    out.write_text(json.dumps(doc, indent=0) + "\n")
    print(f"wrote {out}")


if __name__ == "__main__":
    main()
