"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py full <report.ncu-rep> <out.md>
    python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_bytes.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        stalls = [(k, float(v)) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
                  and v not in ("", "n/a")]
        stalls.sort(key=lambda x: -x[1])
        lines.append("")
        lines.append("Top stall reasons (warps per issue-active cycle):")
        lines.append("")
        for k, v in stalls[:6]:
            lines.append(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.2f}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    im = hdr.index("Metric Name") if "Metric Name" in hdr else None
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])  # launches, us, DRAM MB
    scale_t = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    scale_b = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    for r in data:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0][:70]
        metric = r[im] if im is not None else "gpu__time_duration.sum"
        v = float(r[iv].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v * scale_t.get(r[iu], 1.0)
        elif metric.startswith("dram__bytes"):
            agg[name][2] += v * scale_b.get(r[iu], 1e-6)
    ours = {k: v for k, v in agg.items() if "smp" in k or "cub::" in k or "CUB" in k}
    tot = sum(v[1] for v in ours.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{path}`", "",
             "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.", "",
             f"Library kernels only (data generation excluded): {sum(v[0] for v in ours.values())} launches, {tot:.1f} us", "",
             "| kernel | launches | total us | share | DRAM MB |", "|---|---|---|---|---|"]
    for k, (n, t, mb) in sorted(ours.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% | {mb:.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
