"""Print the key fields of a bench.py JSON line:  python tools/bench_summary.py gpurun_out/bench.log"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
for k in ["value", "ms_per_step", "decode_tok_s", "kv_migration_gbs", "gpu_launches", "clocks"]:
    print(k, d.get(k))
if d.get("e2e"):
    print("e2e", d["e2e"]["value"], d["e2e"].get("probes"))
r = d.get("roofline") or {}
print("roof", {k: r.get(k) for k in ["kernel", "achieved", "frac", "share_of_step", "avg_launch_ms"]})
for n, r in (d.get("roofline_other_kernels") or {}).items():
    print(" ", n, {k: r.get(k) for k in ["achieved", "frac", "share_of_step", "avg_launch_ms"]})
for p in d.get("probes", []):
    if isinstance(p, dict):
        print(" probe", round(p["rate"], 1), p["attainment"], round(p["ttft_p90"] or 0, 3),
              round(p["tbt_p90"] or 0, 4), p["batches"])
print("cpu_baseline", d.get("cpu_baseline"))
print("budgets", d.get("config", {}).get("budgets"))
