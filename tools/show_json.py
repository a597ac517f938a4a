"""Print selected keys of a bench JSON line: python tools/show_json.py file key.sub ..."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
for k in sys.argv[2:]:
    v = d
    for part in k.split("."):
        v = v.get(part) if isinstance(v, dict) else None
    print(k, "=", json.dumps(v))
