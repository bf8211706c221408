"""Aggregate an ncu 'cuda,sass' source CSV per CUDA source line: instructions and stall samples."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None; cur = None
inst = collections.Counter(); stall = collections.Counter(); text = {}
stalls = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Function Name": continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]:  # a CUDA source line row
        cur = (fname, int(r[0])); text[cur] = r[1][:80]
    try:
        n = int(r[hdr.index("Instructions Executed")] or 0)
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    if cur is None: continue
    inst[cur] += n; stall[cur] += s
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try: stalls[cur][name[6:]] += int(r[i] or 0)
            except ValueError: pass
ti = sum(inst.values()); ts = sum(stall.values())
print("total inst", ti, "stall samples", ts)
for k, v in sorted(stall.items(), key=lambda x: -x[1])[:top]:
    top3 = ", ".join(f"{a}:{b}" for a, b in stalls[k].most_common(3))
    print(f"stall {v/ts*100:5.1f}% inst {inst[k]/ti*100:5.1f}%  {k[0]}:{k[1]:4d} {text.get(k,'')[:60]:60s} [{top3}]")
