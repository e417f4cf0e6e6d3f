"""Summarise `ncu --set full` captures of the merge kernel into
profiles/<round>_ncu_summary.json and profiles/traffic.json (DRAM bytes read +
written per launch, the bench's roofline.traffic).

    python tools/ncu_summary.py r01 C2=gpurun_out/ncu_C2.ncu-rep C5=... [X=rep@k]
(traffic.json is only updated for the BASELINE config labels C1..C5.)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep, index=0):
    if rep.endswith(".csv"):  # a raw page exported on the GPU box (ncu -i rep --page raw --csv)
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2 + index]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def stalls(d):
    st = {}
    for k, (u, v) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda t: -t[1])[:6]
    return {k: round(100 * x / tot, 1) for k, x in top}


def main():
    rnd = sys.argv[1]
    out_path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.json")
    summary = json.load(open(out_path)) if os.path.exists(out_path) else {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split("=", 1)
        index = 0
        if "@" in rep:  # report@k: the k-th kernel of a multi-kernel capture
            rep, k = rep.rsplit("@", 1)
            index = int(k)
        d, kname = raw(rep, index)
        entry = {"kernel": kname, "report": os.path.basename(rep)}
        for k in KEYS:
            if k in d:
                u, v = d[k]
                entry[k] = f"{u} {v}".strip()
        entry["stall_reasons_pct_top6"] = stalls(d)
        summary[cfg] = entry
        try:
            if not cfg.startswith("C"):
                raise KeyError(cfg)
            rb = float(d["dram__bytes_read.sum"][1].replace(",", "")) * SCALE[d["dram__bytes_read.sum"][0]]
            wb = float(d["dram__bytes_write.sum"][1].replace(",", "")) * SCALE[d["dram__bytes_write.sum"][0]]
            traffic[cfg] = int(rb + wb)
        except (KeyError, ValueError):
            pass
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant "
                        "kernel from one `ncu --set full` capture (profiles/*_ncu_summary.json). "
                        "Writes still dirty in L2 at kernel end are not counted by ncu.")
    json.dump(summary, open(out_path, "w"), indent=1)
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
