"""Summarise a round's GPU profile into profiles/ (tracked).

Inputs (from tools/profile_round.sh, merged into gpurun_out/):
  decode_<R>.ncu-rep   ncu --set full capture of one decode_step_kernel launch
  launches_<R>.csv     ncu gpu__time_duration.sum launch list of the bench command
  bench_<R>.json       the bench line
Outputs:
  profiles/ncu_<R>_<model>.json   key metrics (dram bytes per launch = roofline
                                  `traffic`, duration, throughput, stalls)
  profiles/launches_<R>.csv       the launch list (copied)
  profiles/summary_<R>.md         human-readable summary
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
MODEL = sys.argv[2] if len(sys.argv) > 2 else "llama31_8b"
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
os.makedirs(PROF, exist_ok=True)

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for i, h in enumerate(hdr):
        if h in KEYS:
            v = vals[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[i]
            if u in UNIT:
                x *= UNIT[u]
            elif u == "ms":
                x *= 1e-3
            elif u == "us":
                x *= 1e-6
            elif u == "ns":
                x *= 1e-9
            out[KEYS[h]] = x
    return out


def stall_summary(rep, top=12):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, vals = rows[0], rows[2]
    st = []
    total = 0.0
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            st.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            total += v
    st.sort(reverse=True)
    return [(100.0 * v / total if total else 0.0, h) for v, h in st[:top]]


def main():
    rep = os.path.join(OUT, f"decode_{R}.ncu-rep")
    m = raw_metrics(rep)
    bench = None
    bpath = os.path.join(OUT, f"bench_{R}.json")
    if os.path.exists(bpath):
        for line in open(bpath):
            if line.strip().startswith("{"):
                bench = json.loads(line)
    traffic = m.get("dram_read", 0) + m.get("dram_write", 0)
    algo = bench["roofline"]["algorithmic_bytes_per_launch"] if bench else None
    summary = {
        "round": R, "model": MODEL, "batch": 1, "ctx": 4096,
        "kernel": "ffb200::decode_step_kernel<Shape<4096,14336,128,32,8,1>>",
        "capture": "ncu --set full --import-source on --clock-control none -k regex:decode_step "
                   "-s 3 -c 1 python tools/perf_probe.py --ncu",
        "dram_bytes_per_launch": traffic,
        "algorithmic_bytes_per_launch": algo,
        "traffic_over_algorithmic": traffic / algo if algo else None,
        "metrics": m,
        "top_stalls": [(h, v) for v, h in stall_summary(rep)],
    }
    with open(os.path.join(PROF, f"ncu_{R}_{MODEL}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    lsrc = os.path.join(OUT, f"launches_{R}.csv")
    if os.path.exists(lsrc):
        shutil.copy(lsrc, os.path.join(PROF, f"launches_{R}.csv"))
    # launch-list shares
    shares = {}
    if os.path.exists(lsrc):
        txt = open(lsrc).read()
        start = txt.find('"ID"')
        rows = list(csv.DictReader(io.StringIO(txt[start:])))
        tot = 0.0
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            t = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            t *= {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(unit, 1e-9)
            k = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
            k = k.split("::")[-1] or r["Kernel Name"][:40]
            shares[k] = shares.get(k, 0.0) + t
            tot += t
        shares = {k: (v, v / tot) for k, v in sorted(shares.items(), key=lambda kv: -kv[1])}
    with open(os.path.join(PROF, f"summary_{R}.md"), "w") as f:
        f.write(f"# Profile {R}: {MODEL} bf16 batch 1, 4096-token KV cache, one B200\n\n")
        if bench:
            f.write(f"bench: {bench['value']} ms/token (device), e2e {bench['e2e']['value']} "
                    f"ms/token; roofline achieved {bench['roofline']['achieved']} GB/s = "
                    f"{bench['roofline']['frac']:.3f} of {bench['roofline'].get('peak_kind', 'measured')} {bench['roofline']['peak']} "
                    f"GB/s; variants {bench.get('variants')}; clocks {bench.get('clocks')}\n\n")
        f.write(f"ncu --set full (one launch, replayed; serialised/cold, compare shares not "
                f"absolutes): duration {m.get('duration', 0) * 1e3:.3f} ms, DRAM read "
                f"{m.get('dram_read', 0) / 1e9:.3f} GB, write {m.get('dram_write', 0) / 1e9:.4f} GB "
                f"(traffic / algorithmic = {summary['traffic_over_algorithmic']}), DRAM "
                f"{m.get('dram_pct_of_peak', 0):.1f}% of peak, SM {m.get('sm_pct_of_peak', 0):.1f}%, "
                f"registers {m.get('registers')}, smem {m.get('smem_dynamic')}\n\n")
        f.write("warp state samples (smsp__pcsamp_warps_issue_stalled_*, % of samples):\n\n")
        for h, v in summary["top_stalls"]:
            f.write(f"- {h}: {v:.1f}%\n")
        if shares:
            f.write("\nlaunch list shares (bench command under ncu, gpu__time_duration.sum):\n\n")
            for k, (t, s) in shares.items():
                f.write(f"- {k}: {t * 1e3:.3f} ms total, {s * 100:.1f}%\n")
    print(open(os.path.join(PROF, f"summary_{R}.md")).read())


if __name__ == "__main__":
    main()
