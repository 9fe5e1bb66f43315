"""Summarize the ncu outputs of tools/profile_round.sh into profiles/ (tracked).

    python tools/summarize_profiles.py r01
Writes profiles/<R>_launches.csv (the raw launch list), profiles/<R>_summary.md
and profiles/ncu_traffic.json (dram bytes per sweep launch, read by bench.py).
"""

from __future__ import annotations

import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_csv(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.reader(lines))


def launches(R):
    rows = read_csv(os.path.join(ROOT, "gpurun_out", f"launches_{R}.csv"))
    hdr = rows[0]
    ki, kn, mn, mv = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[int(r[ki])][r[mn]] = float(r[mv].replace(",", ""))
        names[int(r[ki])] = r[kn]
    agg = collections.OrderedDict()
    total = 0.0
    for i in sorted(per):
        t = per[i].get("gpu__time_duration.sum", 0.0)
        b = per[i].get("dram__bytes_read.sum", 0.0) + per[i].get("dram__bytes_write.sum", 0.0)
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += b
        total += t
    return agg, total


def details(R, prefix="sweep"):
    rows = read_csv(os.path.join(ROOT, "gpurun_out", f"{prefix}_details_{R}.csv"))
    hdr = rows[0]
    ki, kn, mn, mv, mu = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread",
            "Achieved Occupancy", "Issue Slots Busy", "SM Frequency", "Compute (SM) Throughput"]
    out = collections.OrderedDict()
    for r in rows[1:]:
        if r[mn] in want:
            out.setdefault((int(r[ki]), r[kn]), {})[r[mn]] = f"{r[mv]} {r[mu]}"
    return out


def raw(R, prefix="sweep"):
    rows = read_csv(os.path.join(ROOT, "gpurun_out", f"{prefix}_raw_{R}.csv"))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        stalls = []
        for k, v in d.items():
            if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        stalls.sort(reverse=True)

        def num(k):
            try:
                return float(d[k].replace(",", "")) * scale.get(units.get(k, ""), 1.0)
            except Exception:
                return None
        out[int(d["ID"])] = {
            "kernel": d["Kernel Name"],
            "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
            "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "inst": num("smsp__inst_executed.sum"),
            "stalls": [(k, round(100 * s / tot, 1)) for s, k in stalls[:6]],
        }
    return out


def main():
    R = sys.argv[1] if len(sys.argv) > 1 else "r01"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    shutil.copy(os.path.join(ROOT, "gpurun_out", f"launches_{R}.csv"),
                os.path.join(ROOT, "profiles", f"{R}_launches.csv"))
    agg, total = launches(R)
    det = details(R)
    rw = raw(R)
    lines = [f"# ncu summary, round {R}", "",
             "## Launch list of `python bench.py --steps 2 --warmup 3` (ncu, cold cache, serialised)", "",
             "| kernel | launches | total ms | share | avg DRAM bytes/launch |", "|---|---|---|---|---|"]
    for name, (cnt, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {cnt} | {t / 1e6:.3f} | {100 * t / total:.1f}% | {b / cnt:.3e} |")
    lines += ["", f"Total device time under ncu: {total / 1e6:.3f} ms", "",
              "## `ncu --set full` of sweep launches (N=30 p=10 fast run)", ""]
    sweep_bytes = []
    for (i, name), m in det.items():
        lines.append(f"### launch {i}: `{name}`")
        for k, v in m.items():
            lines.append(f"- {k}: {v}")
        r = rw.get(i)
        if r:
            tb = (r["dram_read"] or 0) + (r["dram_write"] or 0)
            sweep_bytes.append(tb)
            lines.append(f"- DRAM read+write: {tb:.4e} B (algorithmic {32 * 2 ** n:.4e} B)")
            lines.append(f"- FP64 pipe active: {r['fp64_pipe_pct']}%  smem wavefronts: {r['smem_wavefronts']:.3e}"
                         f"  bank conflicts: {r['bank_conflicts']:.3e}  warp instrs: {r['inst']:.3e}")
            lines.append("- top stalls: " + ", ".join(f"{k} {v}%" for k, v in r["stalls"]))
        lines.append("")
    if os.path.exists(os.path.join(ROOT, "gpurun_out", f"sym_details_{R}.csv")):
        # symmetric half state (tools/prof_sym.py 30 10): 2^29 amplitudes, 32 B each per sweep
        lines += ["## `ncu --set full` of the symmetric half-state schedule (N=30 p=10, 2^29 "
                  "stored amplitudes: launch-control, mirror low-set, merged sweeps)", ""]
        sd, sr = details(R, "sym"), raw(R, "sym")
        for (i, name), m in sd.items():
            lines.append(f"### launch {i}: `{name}`")
            for k, v in m.items():
                lines.append(f"- {k}: {v}")
            r = sr.get(i)
            if r:
                tb = (r["dram_read"] or 0) + (r["dram_write"] or 0)
                lines.append(f"- DRAM read+write: {tb:.4e} B (algorithmic {32 * 2 ** (n - 1):.4e} B "
                             "read+write, half that for the launch-control sweep)")
                lines.append(f"- FP64 pipe active: {r['fp64_pipe_pct']}%  smem wavefronts: "
                             f"{r['smem_wavefronts']:.3e}  bank conflicts: {r['bank_conflicts']:.3e}  "
                             f"warp instrs: {r['inst']:.3e}")
                lines.append("- top stalls: " + ", ".join(f"{k} {v}%" for k, v in r["stalls"]))
            lines.append("")
    with open(os.path.join(ROOT, "profiles", f"{R}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    full = [b for b in sweep_bytes if b > 0]
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    if full:
        traffic[str(n)] = {"dram_bytes_per_launch": max(full), "round": R,
                           "note": "max over captured read+write sweeps (ncu --set full)"}
        json.dump(traffic, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
