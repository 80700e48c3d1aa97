"""Summarise an ncu --set full capture of the tile kernel: throughput,
DRAM bytes, stall reasons and the hottest SASS lines.  Usage:
python tools/ncu_summary.py rep.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "k_tiles"


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("--page", "raw")
h = rows[0]
for r in rows[2:]:
    if kname not in "".join(r):
        continue
    d = dict(zip(h, r))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
    for k in keys:
        print(f"{k:60s} {d.get(k)} {rows[1][h.index(k)] if k in h else ''}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    print("stall samples:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in
                                      sorted(st.items(), key=lambda kv: -kv[1]) if v / tot > 0.01))
    break
src = page("--page", "source", "--print-source", "sass")
# one section per captured kernel: a "Kernel Name" row, a header row, the SASS rows
sect, cur = [], None
for r in src:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
        sect.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for sc in sect:
    if kname not in sc["name"] or len(sc["rows"]) < 2:
        continue
    hh = sc["rows"][0]
    i = hh.index("Warp Stall Sampling (All Samples)")
    data = [r for r in sc["rows"][1:] if len(r) > i and r[i].replace(".", "").isdigit()]
    tot = sum(float(r[i]) for r in data) or 1
    print("hottest SASS (share of stall samples):", sc["name"][:60])
    for r in sorted(data, key=lambda r: -float(r[i]))[:15]:
        print(f"  {float(r[i]) / tot * 100:5.1f}%  {r[1][:100]}")
    break
