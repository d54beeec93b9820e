# one-off wide parity sweep: 120 seeded step configurations (tests/test_gpu_fuzz.py generator,
# another seed) in every precision whose contract applies; worst deviations per precision
set -u
rm -f gpurun_out/fuzz.jsonl
PFC_FUZZ_CASES=120 PFC_FUZZ_SEED=777 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q 2>&1 | tail -3
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/fuzz.jsonl")]
worst = collections.defaultdict(dict)
for r in rows:
    w = worst[r.get("precision")]
    for k, v in r.items():
        if isinstance(v, float) and k not in ("loss", "loss_ref"):
            w[k] = max(w.get(k, 0.0), v)
print("records", len(rows))
for prec, w in worst.items():
    print(prec, {k: f"{v:.2e}" for k, v in sorted(w.items())})
PY
