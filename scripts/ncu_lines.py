"""Per-source-line samples / instructions / top stalls of an ncu report."""
import collections, csv, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source=cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if len(r) > 20 and r[0] == "Line No")
stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
per = collections.defaultdict(lambda: [0, 0, "", collections.Counter()])
cur = None
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) < 8:
        continue
    if r[0] != "":
        if r[0].isdigit():
            cur = (fname, int(r[0])) if "--by-file" in sys.argv else int(r[0])
            per[cur][2] = r[1][:80]
        continue
    if cur is None:
        continue
    try:
        per[cur][0] += int(r[4]); per[cur][1] += int(r[7])
        for c in stall_cols:
            if c < len(r) and r[c].isdigit():
                per[cur][3][hdr[c]] += int(r[c])
    except ValueError:
        pass
tot = sum(v[0] for v in per.values()) or 1
toti = sum(v[1] for v in per.values()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
argv_pos = [a for a in sys.argv[1:] if not a.startswith("--")]
key = 0 if len(sys.argv) > 3 and sys.argv[3] == 'samples' else 1
print(f"samples {tot}  warp-instr {toti}")
for ln, (s, e, src, st) in sorted(per.items(), key=lambda kv: -kv[1][key])[:n]:
    top = ", ".join(f"{k.replace('stall_', '')}:{v}" for k, v in st.most_common(2))
    lab = f"{ln[0][:10]}:{ln[1]}" if isinstance(ln, tuple) else f"{ln:4d}"
    print(f"{lab} {100*s/tot:5.1f}%s {100*e/toti:5.1f}%i {src[:64]:64s} | {top}")
# optional: stall totals over source-line ranges, e.g. --ranges R:985-1230,H:1240-1340
rng = [a for a in sys.argv if a.startswith("--ranges=")]
if rng:
    for part in rng[0].split("=", 1)[1].split(","):
        name, span = part.split(":")
        lo, hi = map(int, span.split("-"))
        agg, ss, ee = collections.Counter(), 0, 0
        for ln, (s, e, src, st) in per.items():
            l0 = ln[1] if isinstance(ln, tuple) else ln
            fmatch = (not isinstance(ln, tuple)) or ("@" not in name) or name.split("@")[1] in ln[0]
            if lo <= l0 <= hi and fmatch:
                agg.update(st); ss += s; ee += e
        top = ", ".join(f"{k.replace('stall_', '')}:{100*v/max(1,ss):.0f}%" for k, v in agg.most_common(6))
        print(f"{name}: {100*ss/tot:.1f}% samples, {100*ee/toti:.1f}% instr | {top}")
