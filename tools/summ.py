"""Print a compact summary of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "unavailable" in d:
        print(d)
        continue
    cfg = d.get("config", {})
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    print(f"{cfg.get('workload', '')[:3]} impl={d.get('impl', 'ours')} value={d['value']:.4g} {d['unit']} "
          f"ms/step={d['ms_per_step']:.3f} frac={rf.get('frac')} e2e={e2e.get('value')} "
          f"launches={d.get('gpu_launches')} clocks={d.get('clocks', {}).get('sm_mhz')}")
    st = d.get("stage_ms_per_step")
    if st:
        print("   stages:", {k: v for k, v in st.items() if v})
