import json, sys
want_u = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for l in sys.stdin:
    try:
        d = json.loads(l)
    except Exception:
        print(l.strip()); continue
    if want_u and d["U"] != want_u:
        continue
    ul, dl = d["ul"], d["dl"]
    print(d["B"], d["U"], d["C"], ul["kernel"], ul["roofline_frac"], dl["roofline_frac"] if isinstance(dl, dict) else "-")
