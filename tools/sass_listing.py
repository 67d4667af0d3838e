"""Write the SASS of the hot kernels (attention, quantize/append) from the in-tree objects to
profiles/ with an opcode histogram on top (evidence that tcgen05 MMA / TMEM / TMA instructions are
what runs: UTCHMMA, LDTM/STTM, UTMALDG/UBLKCP).  usage: python tools/sass_listing.py <tag>"""
import collections, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
objs = {"attention": os.path.join(ROOT, "paper_2605_18739_b200/_build/attention.cu.o"),
        "quant": os.path.join(ROOT, "paper_2605_18739_b200/_build/quant.cu.o")}
want = {"attention": ["attn_ws_kernelILi128ELb1ELb0ELb0ELb0E", "attn_ws_kernelILi128ELb0ELb1ELb0ELb0E", "combine_kernelILi128E"],
        "quant": ["quant_sp_kernelILi0ELi128ELi0E", "quant2_kernelILi0ELi128ELi0E"]}
for name, obj in objs.items():
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    out = []
    for f in funcs[1:]:
        fname = f.split("\n", 1)[0].strip()
        if not any(w in fname for w in want[name]):
            continue
        lines = [l for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
        ins = [re.sub(r"^\s*/\*[0-9a-f]+\*/\s*", "", l).split(";")[0].strip() for l in lines]
        hist = collections.Counter()
        for i in ins:
            t = i.split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            hist[op.split(".")[0]] += 1
        out.append(f"== {fname}\n{len(ins)} instructions; opcode histogram (static):\n" +
                   "\n".join(f"  {k:12s} {v}" for k, v in hist.most_common(45)) + "\n\n" + "\n".join(ins) + "\n")
    path = os.path.join(ROOT, "profiles", f"sass_{name}_{tag}.txt")
    open(path, "w").write("\n".join(out))
    print(path, sum(len(o) for o in out))
