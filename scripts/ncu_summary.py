#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (run here, on the CPU box).
(`full` also reads the raw-page CSV export of a report made on the GPU box.)

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <report.ncu-rep> <config> <alg_bytes_per_launch> <out.json> [kernel-substring]
  python scripts/ncu_summary.py stalls <source-page.csv[.gz]> <config> <out.json> [kernel-substring]
      (warp-stall sampling by reason and the hottest SASS lines, from `ncu -i R --page source
       --csv --print-source sass`, merged into the config's entry)
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    if path.endswith(".gz"):
        import gzip
        lines = gzip.open(path, "rt").read().splitlines()
    else:
        lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        us = v * 1e-3 if u == "ns" else (v if u in ("us", "usecond") else v * 1e3)
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list summary: {path}\n\n")
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare SHARES)\n\n")
        fh.write("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            fh.write(f"| `{k[:80]}` | {cnt[k]} | {v / 1e3:.2f} | {100 * v / T:.1f}% | {v / cnt[k]:.1f} |\n")
    print(open(out).read())


METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
           "sm__cycles_elapsed.avg.per_second"]


def full(rep, config, alg_bytes, out, pick=None):
    """rep: an .ncu-rep, or its `ncu -i ... --page raw --csv` export (.csv / .csv.gz, summarised on the box)."""
    if rep.endswith(".csv.gz"):
        import gzip
        raw = gzip.open(rep, "rt").read()
    elif rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        kname = vals[hdr.index("Kernel Name")]
        if kname in res:
            continue                  # several launches of one kernel: the first
        d = {}
        for m in METRICS:
            if m in hdr:
                d[m] = {"value": vals[hdr.index(m)], "unit": units[hdr.index(m)]}
        res[kname] = d
    def gb(x):
        v = float(x["value"].replace(",", ""))
        return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}[x["unit"]]
    k, d = next((kv for kv in res.items() if pick is None or pick in kv[0]))
    traffic = (gb(d["dram__bytes_read.sum"]) + gb(d["dram__bytes_write.sum"])) * 1e9
    summ = {"kernel": k, "report": rep, "metrics": d, "dram_bytes_per_launch": traffic,
            "alg_bytes_per_launch": float(alg_bytes), "traffic_over_alg": traffic / float(alg_bytes)}
    allp = {}
    try:
        allp = json.load(open(out))
    except Exception:
        pass
    allp[config] = summ
    json.dump(allp, open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1))


def stalls(path, config, out, top=12, pick=None):
    """The source page of the first kernel in the export (or the first whose name contains pick)."""
    import gzip
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    lines = raw.splitlines()
    heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
    sec = 0
    if pick is not None:
        sec = next(k for k in range(len(heads) - 1) if pick in lines[heads[k]])
    lines = lines[heads[sec]:heads[sec + 1]] if len(heads) > 1 else lines
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in rows:
        for c in cols:
            try:
                tot[c] += float(r[ix[c]])
            except ValueError:
                pass
    T = sum(tot.values()) or 1.0
    key = "Warp Stall Sampling (All Samples)"
    hot = sorted(rows, key=lambda r: -float(r[ix[key]] or 0))[:top]
    summ = {"source_page": path, "kernel": lines[0].split(",", 1)[-1].strip().strip(',').strip('"'), "samples": T,
            "by_reason": {c: round(v / T, 3) for c, v in tot.most_common() if v},
            "hottest": [{"sass": r[ix["Source"]].strip(), "samples": float(r[ix[key]] or 0),
                         "reasons": {c: float(r[ix[c]]) for c in cols if r[ix[c]] not in ("0", "")}} for r in hot]}
    allp = {}
    try:
        allp = json.load(open(out))
    except Exception:
        pass
    allp.setdefault(config, {})["stalls"] = summ
    json.dump(allp, open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "stalls":
        stalls(sys.argv[2], sys.argv[3], sys.argv[4], pick=sys.argv[5] if len(sys.argv) > 5 else None)
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5], sys.argv[6] if len(sys.argv) > 6 else None)
