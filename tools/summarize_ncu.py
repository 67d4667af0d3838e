"""Summarise ncu captures of a round into profiles/ (run here, on the CPU box, after gpurun).
usage: python tools/summarize_ncu.py <tag>"""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)
out = [f"# ncu summary, round tag {tag}\n"]

# launch list (cold-cache, serialised: compare shares, not absolutes)
rows = list(csv.reader(open(os.path.join(G, f"launches_{tag}.csv"))))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
per = defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        v = float(d["Metric Value"])
        unit = d.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else v * (1000.0 if unit == "ms" else 1.0)
        tot[name] += v
        cnt[name] += 1
        per[name].append(v)
ours = {k: v for k, v in tot.items() if "kvq" in k or "attn" in k or "quant" in k or "combine" in k}
s = sum(ours.values())
out.append("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 3 --warmup 3)\n")
out.append("| kernel | launches | total us | mean us | median us | share of our kernels |\n|---|---|---|---|---|---|\n")
for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
    med = sorted(per[k])[len(per[k]) // 2]
    out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / cnt[k]:.2f} | {med:.2f} | {100 * v / s:.1f}% |\n")
out.append("\n(The bench fills the window with chunks 0-5 first -- 4,680 to 28,080 keys -- so the attention mean mixes "
           "sizes; the median is the timed 32,760-key step.)\n")

keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]
traffic = {}
for rep, label in ((f"attn_{tag}", "attn_ws_kernel"), (f"quant_{tag}", "quant_sp_kernel")):
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        out.append(f"\n## `{d['Kernel Name'][:90]}` (`ncu --set full`, one launch)\n\n| metric | value |\n|---|---|\n")
        for k in keys:
            if k in d:
                out.append(f"| {k} | {d[k]} {u.get(k, '')} |\n")
        def mb(k):
            v = float(d[k]); un = u.get(k, "")
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(un, 1.0)
        traffic[label] = {"dram_read_MB": mb("dram__bytes_read.sum"), "dram_write_MB": mb("dram__bytes_write.sum"),
                          "bytes": (mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")) * 1e6, "source": rep}


def stall_table(rep, region=None):
    """Warp-stall sampling from the SASS source page: reasons summed over the kernel, and over a
    SASS address range picked by `region` (first..last instruction whose text matches)."""
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        return
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    spans = [("whole kernel", 0, len(data) - 1)]
    if region:
        idx = [i for i, d in enumerate(data) if any(t in d["Source"] for t in region[1])]
        if idx:
            spans.append((region[0], idx[0], idx[-1]))
    for label, lo, hi in spans:
        tot = sum(float(data[i]["Warp Stall Sampling (All Samples)"] or 0) for i in range(lo, hi + 1))
        agg = {r: sum(float(data[i][r] or 0) for i in range(lo, hi + 1)) for r in reasons}
        top = sorted(agg.items(), key=lambda kv: -kv[1])[:8]
        out.append(f"\n### {rep}: warp-stall samples, {label} ({int(tot)} samples)\n\n| reason | share |\n|---|---|\n")
        for r, v in top:
            out.append(f"| {r} | {100 * v / max(tot, 1):.1f}% |\n")


stall_table(f"attn_{tag}", ("softmax max/exp/sum region (FMNMX3 .. FHADD)", ("FMNMX3", "MUFU.EX2", "FHADD")))
stall_table(f"quant_{tag}")
out.append("\n(Samples count every resident warp, including warps parked on mbarrier waits (BRA spin) "
           "or at EXIT, so the whole-kernel shares mix roles; the region row isolates the softmax loop.)\n")
open(os.path.join(P, f"ncu_summary_{tag}.md"), "w").write("".join(out))
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
os.system(f"cp {os.path.join(G, f'launches_{tag}.csv')} {os.path.join(P, f'launches_{tag}.csv')}")
print("".join(out))
