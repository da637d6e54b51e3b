"""Summarise an ncu report: duration, DRAM bytes, IPC, stall reasons, dynamic SASS mix (dev tool)."""
import csv, collections, re, subprocess, sys, io

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
d = data[0]
def g(name):
    try:
        return d[hdr.index(name)]
    except ValueError:
        return "?"
print("dur_ms", g("gpu__time_duration.sum"), "dram_rd", g("dram__bytes_read.sum"), "dram_wr", g("dram__bytes_write.sum"),
      "inst", g("smsp__inst_executed.sum"), "regs", g("launch__registers_per_thread"),
      "ipc", g("sm__inst_executed.avg.per_cycle_active"))
# amplitudes per launch: argv[2], else from the DRAM read bytes in GB (one read of a complex64 state)
try:
    amps = float(sys.argv[2]) if len(sys.argv) > 2 else float(g("dram__bytes_read.sum")) * 1e9 / 8
except ValueError:
    amps = 2**28
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            st.append((float(d[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st)
print("stalls:", ", ".join(f"{h} {v/tot*100:.1f}%" for v, h in sorted(st, reverse=True)[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex, sw = collections.Counter(), collections.Counter()
nk = 0
for r in rows:
    if r and r[0] == "Kernel Name":
        nk += 1
        continue
    if nk != 1 or len(r) <= iE:
        continue
    try:
        e, s = int(r[iE] or 0), int(r[iW] or 0)
    except ValueError:
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    if m:
        ex[m.group(2)] += e
        sw[m.group(2)] += s
tot = sum(ex.values())
tots = sum(sw.values()) or 1
print(f"warp instr {tot}  per amp {tot*32/amps:.1f}")
for op, e in ex.most_common(22):
    print(f"  {op:10s} {e/tot*100:5.1f}%  {e*32/amps:6.2f}/amp  stall {sw[op]/tots*100:5.1f}%")
