"""Summarise an ncu launch list (ncu --metrics gpu__time_duration.sum --csv --log-file X) of
bench.py: the kernels of the last step (from the last sampler_kernel through the next dW
GEMM), their times and their shares of the serialised sum.
Usage: python profiles/launch_summary.py <launches.csv> [header line ...]"""
import csv
import sys


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r["Metric Unit"]
            us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
            rows.append((r["Kernel Name"], us))
    starts = [i for i, (k, _) in enumerate(rows) if k.startswith("mark_kernel")]
    if not starts:
        sys.exit("no mark_kernel in the launch list")
    i0 = starts[-1]
    step = []
    for k, us in rows[i0:]:
        step.append((k, us))
        if "DwUpdateEpi" in k or "dw_rows_update" in k:
            break
    total = sum(us for _, us in step)
    for h in sys.argv[2:]:
        print(h)
    print(f"last step's launches ({len(step)} kernels; share of the serialised sum in brackets):")
    for k, us in step:
        print(f"  {us:9.2f} us  [{100 * us / total:5.1f}%]  {k[:100]}")
    print(f"  {total:9.2f} us  total (bench, graph replay, warm: see BENCH line ms_per_step)")


if __name__ == "__main__":
    main()
