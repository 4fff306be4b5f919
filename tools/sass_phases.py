"""Per-phase instruction / stall attribution for a kernel in an ncu report.

usage: python tools/sass_phases.py <rep> <mangled-substring> <file> lo:hi:name ... [--per N]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kname, fname = sys.argv[1], sys.argv[2], sys.argv[3]
per = 1.0
args = sys.argv[4:]
if "--per" in args:
    i = args.index("--per"); per = float(args[i + 1]); args = args[:i] + args[i + 2:]
phases = [(int(a.split(":")[0]), int(a.split(":")[1]), a.split(":")[2]) for a in args]
so = os.path.abspath("paper_2305_15661_b200/_strom_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
dis = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    d = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if kname in d:
        dis = d
        break
a2l, a2op, cur, infun = {}, {}, None, False
for ln in dis.splitlines():
    if ln.startswith("//---------------------"):
        infun = kname in ln; continue
    if not infun: continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m: cur = (m.group(1), int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
    if m and cur:
        a = int(m.group(1), 16); a2l[a] = cur; a2op[a] = m.group(3).split(".")[0]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); hdr = rows[1]
ia, iex, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0.0, 0.0]); ops = collections.Counter(); base = None; tot = 0.0
for r in rows[2:]:
    try: a = int(r[ia], 16); ex = float(r[iex] or 0); sm = float(r[isamp] or 0)
    except (ValueError, IndexError): continue
    base = a if base is None else base; a -= base
    f, l = a2l.get(a, ("?", 0)); tot += ex
    ph = f
    if f == fname:
        for lo, hi, n in phases:
            if lo <= l <= hi: ph = n
    agg[ph][0] += ex; agg[ph][1] += sm; ops[a2op.get(a, "?")] += ex
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} inst/unit={v[0] / per:8.0f} ({100 * v[0] / tot:4.1f}%)  stall-samples {100 * v[1] / ts:4.1f}%")
print("total inst/unit", tot / per)
print(" ".join(f"{op}:{c / per:.0f}" for op, c in ops.most_common(24)))
