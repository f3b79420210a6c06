"""Summarise an ncu --set full report into profiles/ (markdown + traffic JSON).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_full.md [profiles/ncu_traffic.json]
"""
import csv, io, json, subprocess, sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "local_load_bytes", "smsp__sass_inst_executed_op_local_ld.sum",
    "sm__inst_executed.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


# kernel → bench.py kernel class (vc_profile classes)
CLASS = {"primary": "primary", "rings": "rings", "wave_scan": "wave_scan", "gather": "gather",
         "gather_emit": "gather", "gather_occl": "gather", "gather_eval": "gather", "gather_occl_pt": "gather",
         "gather_delta": "gather", "gather_delta_pt": "gather", "delta_single": "assemble", "primary_pt": "primary",
         "directions": "primary", "delaunay_smem": "delaunay", "delaunay_retry": "delaunay",
         "delaunay_hull": "delaunay", "delaunay_cap": "delaunay", "delaunay_capg": "delaunay", "cap_bin": "delaunay", "delaunay_warp": "delaunay", "delaunay_list": "delaunay",
         "delaunay_rest": "delaunay", "assemble_t": "assemble", "asm_eval": "assemble",
         "tri_compact": "tri_compact", "own_scan": "tri_compact", "tri_scatter": "tri_compact", "degree": "degree", "live_masks": "assemble", "assemble": "assemble",
         "asm_final": "assemble", "make_record": "make_record", "seedseq": "seedseq", "march": "march",
         "interpolate": "interpolate"}


def main():
    rep, md = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[3] if len(sys.argv) > 3 else None
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{rep}`", "", "| kernel | metric | value | unit |", "|---|---|---|---|"]
    traffic = {}
    stalls = {}
    for row in rows:
        name = row[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        for m in METRICS:
            if m in col and row[col[m]] not in ("", "n/a"):
                lines.append(f"| {short} | {m} | {row[col[m]]} | {units[col[m]]} |")
        rb = to_bytes(row[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wb = to_bytes(row[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        key = short.replace("vc::", "").replace("k_", "").split("<")[0]
        traffic[key] = traffic.get(key, 0.0) + rb + wb  # summed over launches (window classes)
        st = []
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    st.append((float(row[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        stalls[short] = [(n, round(v / tot, 3)) for v, n in sorted(st, reverse=True)[:6]]
    lines += ["", "## Warp stall reasons (pc sampling share)", ""]
    for k, v in stalls.items():
        lines.append(f"- {k}: " + ", ".join(f"{n} {s:.1%}" for n, s in v))
    lines += ["", "## DRAM traffic per launch (read + write bytes)", ""]
    for k, v in traffic.items():
        lines.append(f"- {k}: {v:.4g} B")
    open(md, "w").write("\n".join(lines) + "\n")
    if traffic_out:
        per_class = {}
        for k, v in traffic.items():
            c = CLASS.get(k)
            if c:
                per_class[c] = per_class.get(c, 0.0) + v
        inst = defaultdict(float)  # warp instructions per class over the captured launches
        for row in rows:
            short = row[col["Kernel Name"]].split("(")[0].replace("void ", "")
            key = short.replace("vc::", "").replace("k_", "").split("<")[0]
            c = CLASS.get(key)
            for m in ("sm__inst_executed.sum", "smsp__inst_executed.sum"):
                if c and m in col and row[col[m]] not in ("", "n/a"):
                    inst[c] += float(row[col[m]].replace(",", ""))
                    break
        json.dump({"report": rep, "per_kernel": traffic, "per_class": per_class, "inst_per_class": dict(inst)},
                  open(traffic_out, "w"), indent=1)
    print(open(md).read())


if __name__ == "__main__":
    main()
