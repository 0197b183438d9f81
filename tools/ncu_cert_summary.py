"""Summarise an `ncu --set full` capture of k_cert_dense launches (tools/prof_cert.py, two
certified solves) against the certified pass's byte model:
    per full layer t: 4 * key_space (rank entries) + 28 * n_t (value 8 + action 4 + pair 16
    written) + 16 * n_{t+1} (successor pairs read once).

    python tools/ncu_cert_summary.py report.ncu-rep tools/c4_layers.json <first_skip> out.json"""
import csv
import io
import json
import subprocess
import sys


def main(rep, layers_json, skip, out):
    lay = json.loads(open(layers_json).read())
    order = lay["dense_layers_desc"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}
    launches = []
    for j, r in enumerate(rows[2:]):
        t = order[(skip + j) % len(order)]
        n, n1 = lay["layers"][t], lay["layers"][t + 1]
        alg = 4 * lay["key_space"] + 28 * n + 16 * n1
        g = lambda k: float(r[hdr.index(k)].replace(",", "")) * scale.get(units[hdr.index(k)], 1)  # noqa: E731
        dram = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        tt = float(r[hdr.index("gpu__time_duration.sum")].replace(",", "")) * tscale[units[hdr.index("gpu__time_duration.sum")]]
        pick = lambda k: float(r[hdr.index(k)].replace(",", ""))  # noqa: E731
        launches.append({
            "layer": t, "states": n, "key_space": lay["key_space"], "alg_bytes": alg,
            "dram_bytes": dram, "dram_over_alg": dram / alg, "ncu_time_us": tt * 1e6,
            "dram_GBps": dram / tt / 1e9, "alg_GBps": alg / tt / 1e9,
            "l2_hit_pct": pick("lts__t_sector_hit_rate.pct"),
            "l2_bytes": 32.0 * pick("lts__t_sectors.sum") if "lts__t_sectors.sum" in hdr else None,
            "warps_active_pct": pick("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pick("smsp__issue_active.avg.pct_of_peak_sustained_active")})
    doc = {"kernel": "k_cert_dense (certified pass, key-space walk)", "workload": lay["workload"],
           "capture": f"ncu --set full --clock-control none, launches {skip}.. of tools/prof_cert.py",
           "dram_bytes_per_launch": launches[0]["dram_bytes"],
           "alg_bytes_per_launch": launches[0]["alg_bytes"], "launches": launches,
           "note": "dram/alg = %.2f on layer %d" % (launches[0]["dram_over_alg"], launches[0]["layer"])}
    open(out, "w").write(json.dumps(doc, indent=1))
    print(json.dumps(doc, indent=1)[:2500])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4])
