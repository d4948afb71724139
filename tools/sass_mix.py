"""Dynamic SASS opcode mix (warp-level instructions executed) and stall
samples per opcode from an ncu --page source --print-source sass CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_src, i_exec, i_samp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt = collections.Counter()
samp = collections.Counter()
for r in rows[2:]:
    if len(r) <= i_exec:
        continue
    op = r[i_src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    try:
        cnt[o] += int(r[i_exec] or 0)
        samp[o] += int(r[i_samp] or 0)
    except ValueError:
        pass
tot = sum(cnt.values())
ts = sum(samp.values())
print(f"total warp-instructions {tot}  stall samples {ts}")
for o, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {c:12d} {100 * c / tot:5.1f}%   samples {100 * samp[o] / max(ts, 1):5.1f}%")
