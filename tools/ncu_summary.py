"""Summarise an ncu --set full capture of k_wave_layer or k_cert_dense (C4,
tools/prof_sweep.py) into profiles/ncu_{wave,cert}.json: per captured launch, DRAM traffic vs
the algorithmic bytes of that layer.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep <first_skip> [out.json] [wave|cert]

`first_skip` is the -s value used for the capture: layer launches are numbered over solves of
H=48 layer launches each (cert: the full layers only), layers descending (t = H-1 .. 0)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(rep, skip, out=None, kind="wave"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lay = json.loads((ROOT / "tools" / "c4_layers.json").read_text())
    H = lay["H"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    full = 531441  # C4 layer key space (9^6)
    # cert: k_cert_dense runs the full layers (at least half of the key space reached)
    order = [t for t in range(H - 1, -1, -1) if kind != "cert" or (t >= 1 and 2 * lay["layers"][t]["n"] >= full)]
    if kind == "sweep":  # Jacobi with the layer skip: sweep k = 1..H+1 covers layers 0..H-k+1
        order = list(range(1, H + 2))
    for j, r in enumerate(rows[2:]):
        t = order[(skip + j) % len(order)]
        if kind == "sweep":
            k = t
            last = min(H, H - k + 1)
            rows_k = sum(x["n"] for x in lay["layers"][:last + 1])
            edges_k = sum(x["edges"] for x in lay["layers"][:last + 1])
            g = lambda name: float(r[hdr.index(name)]) * scale.get(units[hdr.index(name)], 1)
            dram = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
            tu = units[hdr.index("gpu__time_duration.sum")]
            tt = float(r[hdr.index("gpu__time_duration.sum")]) * (1e-6 if tu == "us" else 1e-3 if tu == "ms" else 1e-9)
            alg = 24 * rows_k + 12 * edges_k  # 24 + 12*E/S bytes per backup
            launches.append({"sweep": k, "rows": rows_k, "edges": edges_k, "alg_bytes": alg,
                             "dram_bytes": dram, "dram_over_alg": dram / alg,
                             "ncu_time_us": tt * 1e6, "dram_GBps": dram / tt / 1e9,
                             "l2_hit_pct": float(r[hdr.index("lts__t_sector_hit_rate.pct")]),
                             "warps_active_pct": float(r[hdr.index("sm__warps_active.avg.pct_of_peak_sustained_active")]),
                             "issue_active_pct": float(r[hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")])})
            continue
        n, e = lay["layers"][t]["n"], lay["layers"][t]["edges"]
        n_next = lay["layers"][t + 1]["n"]
        m = H - t
        # per layer: row_ptr 4 + value 8 + action 4 + winner's action 4 per state, succ 4 +
        # reward 8 per edge, versions written (8 per backup) and the successor versions read
        # once (8 * n_{t+1} * (m-1))
        alg = 20 * n + 12 * e + 8 * n * m + 8 * n_next * (m - 1)
        if kind == "cert":
            # k_cert_dense (pairs by key-space index, a thread per key-space index): the rank
            # entry of every index 4, per state value 8 + action 4 + pair written 16, the
            # successors' pairs read once (16 * n_{t+1})
            alg = 4 * full + 28 * n + 16 * n_next
        g = lambda k: float(r[hdr.index(k)]) * scale.get(units[hdr.index(k)], 1)
        dram = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        tt = float(r[hdr.index("gpu__time_duration.sum")]) * (1e-6 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1e-9)
        launches.append({"layer": t, "states": n, "edges": e, "versions": m,
                         "alg_bytes": alg, "dram_bytes": dram, "dram_over_alg": dram / alg,
                         "ncu_time_us": tt * 1e6, "dram_GBps": dram / tt / 1e9,
                         "l2_hit_pct": float(r[hdr.index("lts__t_sector_hit_rate.pct")]),
                         "warps_active_pct": float(r[hdr.index("sm__warps_active.avg.pct_of_peak_sustained_active")]),
                         "issue_active_pct": float(r[hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")])})
    summary = {"kernel": {"cert": "k_cert_dense<1,false,3>", "sweep": "k_sweep<false>"}.get(kind, "k_wave_layer<false>"),
               "capture": f"ncu --set full, C4, launches {skip}..{skip + len(launches) - 1} of tools/prof_sweep.py",
               "dram_bytes_per_launch": launches[0]["dram_bytes"],
               "alg_bytes_per_launch": launches[0]["alg_bytes"], "launches": launches,
               "note": "dram/alg = %.2f on %s %d" % (launches[0]["dram_over_alg"], "sweep" if kind == "sweep" else "layer",
                                                     launches[0]["sweep" if kind == "sweep" else "layer"])}
    Path(out or ROOT / "profiles" / f"ncu_{kind}.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else None,
         sys.argv[4] if len(sys.argv) > 4 else "wave")
