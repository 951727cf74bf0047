"""Summarise an ncu SASS source page (csv): top instructions by stall samples,
and total samples / executed instructions per opcode class."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def f(x):
    try: return float(x)
    except: return 0.0
tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(f(d["Instructions Executed"]) for d in data)
print(f"instructions {len(data)}  samples {tot_s:.0f}  executed {tot_i:.0f}")
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter(); aggi = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"] else "?"
    if op.startswith("@"): op = d["Source"].split()[1]
    op = op.split(".")[0]
    agg[op] += f(d["Warp Stall Sampling (All Samples)"]); aggi[op] += f(d["Instructions Executed"])
print("by opcode (samples%, exec%):")
for op, s in agg.most_common(14):
    print(f"  {op:10s} {100*s/tot_s:6.2f}% {100*aggi[op]/tot_i:6.2f}%")
st = collections.Counter()
for d in data:
    for c in stall_cols: st[c] += f(d[c])
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/tot_s:.1f}%" for k, v in st.most_common(8)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top instructions:")
for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:n]:
    top = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"  {d['Address']:>6} {f(d['Warp Stall Sampling (All Samples)']):7.0f} ex={f(d['Instructions Executed']):9.0f} {d['Source'][:60]:60s} {top}")
