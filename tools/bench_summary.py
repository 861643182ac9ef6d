"""Print the headline fields of bench.py JSON lines: python tools/bench_summary.py <file.json>..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f, d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"].get("reasons"),
              d["roofline"]["frac"], "e2e", d.get("e2e", {}).get("value"),
              "accept", json.dumps(k.get("accept")), "compact", json.dumps(k.get("compact")))
    except Exception as e:   # noqa: BLE001
        print(f, "ERR", e)
