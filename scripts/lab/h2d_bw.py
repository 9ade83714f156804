"""Lab: pinned host -> device bandwidth for the e2e step's 585 MB, one copy
stream vs several concurrent copy streams, chunked."""
import json
import torch

dev = torch.device("cuda", 0)
nb = 584908800
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device=dev)
out = {}
for nst in (1, 2, 4):
    for nch in (1, 8, 32):
        if nch < nst:
            continue
        sts = [torch.cuda.Stream(dev) for _ in range(nst)]
        cs = nb // nch

        def run():
            for i in range(nch):
                with torch.cuda.stream(sts[i % nst]):
                    d[i * cs:(i + 1) * cs].copy_(h[i * cs:(i + 1) * cs], non_blocking=True)
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for s in sts:
            s.wait_stream(cur)
        for _ in range(5):
            run()
        for s in sts:
            cur.wait_stream(s)
        b.record(cur)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        out[f"streams{nst}_chunks{nch}"] = round(nb / (ms * 1e-3) / 1e9, 2)
print(json.dumps(out))
