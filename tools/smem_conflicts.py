"""Per-source-line shared-memory excess wavefronts (bank conflicts) from an ncu report.

usage: python tools/smem_conflicts.py <report.ncu-rep> <kernel mangled-name substring> [so]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kname = sys.argv[1], sys.argv[2]
so = sys.argv[3] if len(sys.argv) > 3 else "paper_2305_15661_b200/_strom_b200.so"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
dis = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    d = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if kname in d:
        dis = d
        break
addr2line, cur, infun = {}, None, False
for ln in dis.splitlines():
    if ln.startswith("//---------------------"):
        infun = kname in ln
        continue
    if not infun:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, iex, iw, iid = (hdr.index(k) for k in ("Address", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"))
per = collections.defaultdict(lambda: [0.0, 0.0])
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    line = addr2line.get(a - base, "?")
    per[line][0] += float(r[iex] or 0)
    per[line][1] += float(r[iw] or 0)
tot = sum(v[0] for v in per.values())
print(f"total excessive wavefronts {tot:.3g}")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", 20))]:
    print(f"{100 * v[0] / max(tot, 1):5.1f}%  {k:28s} excess={v[0]:.3g} wavefronts={v[1]:.3g}")
