"""Attribute ncu per-instruction stall samples to CUDA source lines.

usage: python tools/sass_lines.py <report.ncu-rep> <kernel mangled-name substring> [so]
Maps SASS addresses to source lines with `nvdisasm -g` on the cubin embedded
in the library (built with -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
so = sys.argv[3] if len(sys.argv) > 3 else "paper_2305_15661_b200/_strom_b200.so"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
dis = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    kfile = os.environ.get("KFILE")  # attribute inlined code to its call site in this file
    d = subprocess.run(["nvdisasm", "-gi" if kfile else "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if kname in d:
        dis = d
        break
addr2line, cur_line, infun = {}, None, False
for ln in dis.splitlines():
    if ln.startswith("//---------------------"):
        infun = kname in ln
        continue
    if not infun:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m:
        cur_line = f"{m.group(1)}:{m.group(2)}"
        if kfile:
            for fn, li in re.findall(r'"[^"]*?/([^/"]+)", line (\d+)', ln):
                if fn == kfile:
                    cur_line = f"{fn}:{li}"
                    break
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line:
        addr2line[int(m.group(1), 16)] = cur_line
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, isamp, iexec = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
per = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot = 0
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
        base = a if base is None else base
        a -= base
        s = float(r[isamp] or 0)
        ex = float(r[iexec] or 0)
    except (ValueError, IndexError):
        continue
    line = addr2line.get(a, "?")
    per[line][0] += s
    per[line][1] += ex
    for i in stall_cols:
        v = float(r[i] or 0)
        if v:
            per[line][2][hdr[i][6:]] += v
    tot += s
src = {}
top = sorted(per.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", 40))]
for line, (s, ex, st) in top:
    why = ", ".join(f"{k}:{int(v)}" for k, v in st.most_common(3))
    print(f"{100 * s / tot:5.1f}%  {line:28s} inst={ex:.3g}  {why}")
