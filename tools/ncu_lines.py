"""Attribute an ncu SASS profile (executed instructions, stall samples) to
fused.cu source lines via nvdisasm line info (dev tool).
usage: python tools/ncu_lines.py REPORT.ncu-rep CUBIN FUNCTION_SUBSTRING"""
import collections, csv, io, re, subprocess, sys

rep, cubin, fsub = sys.argv[1:4]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
line_of, cur, inside = {}, None, False
for ln in dis:
    if ln.startswith("\t.text.") or ln.startswith(".text."):
        inside = fsub in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m:
        cur = int(m.group(1))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iA, iE, iW = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base, ex, st, nk = None, collections.Counter(), collections.Counter(), 0
for r in rows:
    if r and r[0] == "Kernel Name":
        nk += 1
        continue
    if nk != 1 or len(r) <= iE:
        continue
    try:
        a, e, w = int(r[iA], 16), int(r[iE] or 0), int(r[iW] or 0)
    except ValueError:
        continue
    base = a if base is None else base
    ln = line_of.get(a - base, -1)
    ex[ln] += e
    st[ln] += w
te, ts = sum(ex.values()), sum(st.values())
text = open("paper_2504_03967_b200/csrc/fused.cu").read().split("\n")
print(f"total warp instr {te}")
for ln, e in ex.most_common(40):
    s = text[ln - 1].strip()[:70] if ln > 0 else "?"
    print(f"{ln:5d} {e / te * 100:5.1f}% instr  {st[ln] / ts * 100:5.1f}% stall  {s}")
