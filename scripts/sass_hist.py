"""Summarise an ncu '--page source --csv --print-source sass' dump: instruction mix by opcode,
executed counts, stall samples and shared-memory wavefront excess (for profiles/ notes)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
ops = defaultdict(lambda: [0, 0, 0, 0, 0])
tot_exec = tot_samp = 0
top = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ex = int(r[idx["Instructions Executed"]] or 0)
    sm = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    wf = int(r[idx["L1 Wavefronts Shared"]] or 0)
    wfi = int(r[idx["L1 Wavefronts Shared Ideal"]] or 0)
    ops[op][0] += ex
    ops[op][1] += sm
    ops[op][2] += wf
    ops[op][3] += wfi
    tot_exec += ex
    tot_samp += sm
    top.append((sm, src, ex))
print(f"total executed warp-instr {tot_exec}, stall samples {tot_samp}")
for op, (ex, sm, wf, wfi, _) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{op:10s} exec {ex:9d} ({100*ex/max(tot_exec,1):5.1f}%)  stall-samples {sm:7d} ({100*sm/max(tot_samp,1):5.1f}%)  smem wf {wf} ideal {wfi}")
print("--- top stall lines")
for sm, src, ex in sorted(top, reverse=True)[:25]:
    print(f"{sm:7d} {ex:8d}  {src[:90]}")
