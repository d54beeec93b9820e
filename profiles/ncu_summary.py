"""Summarise an ncu report (raw page + per-opcode SASS stall attribution) into text.
Usage: python profiles/ncu_summary.py <report.ncu-rep> [--sass]"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.sum", "lts__t_bytes.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    # this ncu build's names for the north star's evidence: achieved DRAM bandwidth and
    # tensor-pipe activity (the bench line's gemm_tensor_util is the FLOP-based figure)
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        ent = {"kernel": d["Kernel Name"][:100]}
        for m in METRICS:
            if m in d:
                ent[m] = f"{d[m]} {units[hdr.index(m)]}"
        st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(d[h] or 0)
              for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
        ent["top_stalls"] = sorted(st.items(), key=lambda x: -x[1])[:6]
        res.append(ent)
    return res


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kern, hdr, per = None, None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "Kernel Name":
            kern, hdr = r[1], None
            per[kern] = []
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if kern and hdr and len(r) == len(hdr):
            per[kern].append(dict(zip(hdr, r)))
    res = {}
    for k, v in per.items():
        ops, st = collections.Counter(), collections.Counter()
        for d in v:
            toks = d["Source"].strip().split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            ops[op] += int(d.get("Instructions Executed") or 0)
            st[op] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
        tot, tst = sum(ops.values()) or 1, sum(st.values()) or 1
        res[k[:100]] = {"executed_pct": [(o, round(c / tot * 100, 1)) for o, c in ops.most_common(10)],
                        "stall_samples_pct": [(o, round(c / tst * 100, 1)) for o, c in st.most_common(10)]}
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    for e in raw(rep):
        print(e["kernel"])
        for k, v in e.items():
            if k != "kernel":
                print(f"   {k}: {v}")
    if "--sass" in sys.argv:
        for k, v in sass(rep).items():
            print(k)
            print("   executed:", v["executed_pct"])
            print("   stalls:  ", v["stall_samples_pct"])
