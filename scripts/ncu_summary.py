"""Summarise ncu --set full reports into the profiles/ JSON format.
usage: python scripts/ncu_summary.py out.json name=report.ncu-rep[:problems:alg_bytes_per_problem] ...
Reads `ncu -i <rep> --page raw --csv` (works without a GPU)."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "kernel": "Kernel Name",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_read_pct_of_peak": "dram__bytes_read.sum.pct_of_peak_sustained_elapsed",
    "mem_pct_of_peak": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "duration": "gpu__time_duration.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "block": "launch__block_size",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
    "sm_clock": "sm__cycles_elapsed.avg.per_second",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return v


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for row in data:
        r = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        d = {}
        for k, m in WANT.items():
            if m in r:
                d[k] = _num(r[m])
                if k in ("dram_read", "dram_write"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(m, "byte"), 1)
                    d[k] = d[k] * scale
                if k == "duration":
                    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                             "msecond": 1e3}[u.get(m, "ns")]
                    d["duration_us"] = d.pop(k) * scale
                if k == "sm_clock":
                    scale = {"Ghz": 1.0, "GHz": 1.0, "Mhz": 1e-3, "MHz": 1e-3, "cycle/nsecond": 1.0}[u.get(m, "Ghz")]
                    d["sm_clock_GHz"] = d.pop(k) * scale
        stalls = {k[len(STALL_PREFIX):-len(STALL_SUFFIX)]: _num(v) for k, v in r.items()
                  if k.startswith(STALL_PREFIX) and k.endswith(STALL_SUFFIX) and "not_issued" not in k}
        stalls = {k: v for k, v in stalls.items() if isinstance(v, float)}
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        res.append(d)
    return res


def main():
    out_path = sys.argv[1]
    summary = {}
    for arg in sys.argv[2:]:
        name, spec = arg.split("=", 1)
        parts = spec.split(":")
        rep = parts[0]
        try:
            launches = summarise(rep)
        except Exception as e:  # a capture that did not happen: say so, keep the others
            summary[name] = {"error": str(e)[:200]}
            continue
        d = launches[0]
        if len(parts) >= 3:
            problems, per = int(parts[1]), float(parts[2])
            d["problems"] = problems
            d["alg_bytes"] = problems * per
            d["dram_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
            d["dram_bytes_per_problem"] = round(d["dram_bytes"] / problems, 1)
            if "duration_us" in d:
                d["alg_GBps_at_ncu_duration"] = round(d["alg_bytes"] / (d["duration_us"] * 1e-6) / 1e9, 1)
                d["dram_GBps_at_ncu_duration"] = round(d["dram_bytes"] / (d["duration_us"] * 1e-6) / 1e9, 1)
        summary[name] = d
    json.dump(summary, open(out_path, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
