"""Summarise ncu captures into profiles/ (committed evidence).

  python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <round tag>
writes profiles/<tag>_kernels.md, profiles/<tag>_launches.csv (per-launch device times)
and updates profiles/traffic.json (dram bytes per launch of each kernel).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main(rep, launches, tag):
    rows = raw(rep)
    lines = [f"# ncu summary {tag}", "", f"source: `{os.path.basename(rep)}` "
             "(ncu --set full --clock-control none; per-launch numbers are cold-cache and serialised)", ""]
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    seen = set()
    for d, u in rows:
        name = d.get("Kernel Name", "?")
        # lcsf::kernel<attn_fwd_template<128, 1, 0>> -> attn_fwd_template<128, 1, 0>
        inner = name.split("kernel<", 1)[1] if name.startswith("void kernel<") or "::kernel<" in name else name
        base = inner.split("(")[0].replace("void ", "")
        short = base.split("::")[-1].split("<")[0]
        key = f"{short}<{base.split('<')[1].split('>')[0]}>" if "<" in base else short
        if key in seen:
            continue
        seen.add(key)
        lines += [f"## {key}", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in d:
                lines.append(f"| {label} (`{m}`) | {d[m]} {u.get(m, '')} |")
        try:
            b = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
                to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            traffic[short] = b
            lines.append(f"| dram read+write bytes per launch | {b:.4g} |")
        except Exception:
            pass
        lines.append("")
    with open(os.path.join(ROOT, "profiles", f"{tag}_kernels.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)
    # per-launch device times
    out = []
    reader = list(csv.reader(open(launches)))
    hdr = None
    for r in reader:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            dd = dict(zip(hdr, r))
            if dd.get("Metric Name") == "gpu__time_duration.sum":
                out.append((dd["ID"], dd["Kernel Name"][:90], dd["Metric Value"], dd["Metric Unit"]))
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "gpu__time_duration.sum", "unit"])
        w.writerows(out)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main(*sys.argv[1:4])
