"""Print the headline and per-stage milliseconds of bench.py JSON lines (files given on argv)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    st = d.get("stages") or {}
    ms = {k: round(v["ms_per_step"], 3) for k, v in st.items() if isinstance(v, dict)}
    e2e = (d.get("e2e") or {}).get("value")
    print(f, round(d["value"], 2), d["unit"], "ms/step", round(d["ms_per_step"], 3), "e2e", e2e,
          "frac", (d.get("roofline") or {}).get("frac"), ms)
