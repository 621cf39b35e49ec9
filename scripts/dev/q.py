import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["steps"], round(d["value"],3), round(d["ms_per_step"],2), (d.get("e2e") or {}).get("value"))
