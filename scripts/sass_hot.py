"""Group SASS lines of an ncu report by equal execution count; print the blocks with most stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = hdr.index('Instructions Executed'); src = hdr.index('Source'); st = hdr.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[2:]:
    try: n = int(r[ix] or 0)
    except ValueError: continue
    data.append((int(r[0], 16), n, r[src], int(r[st] or 0)))
base = data[0][0]
groups = []; cur = None
for a, n, s, stl in data:
    if cur and cur[1] == n:
        cur[2] += 1; cur[3] += n; cur[5] += stl; cur[6].append((stl, s))
    else:
        if cur: groups.append(cur)
        cur = [a - base, n, 1, n, s, stl, [(stl, s)]]
groups.append(cur)
tot = sum(g[3] for g in groups); ts = sum(g[5] for g in groups)
print('total instr %.1fM stall samples %d' % (tot / 1e6, ts))
for g in sorted(groups, key=lambda g: -g[5])[:top]:
    worst = max(g[6])
    print(f"off {g[0]:6x} count {g[1]:>10} ninstr {g[2]:>4} instr {g[3]/1e6:8.2f}M stalls {g[5]:>7} ({100*g[5]/ts:4.1f}%) first: {g[4][:40]:40s} worst: {worst[1][:50]} ({worst[0]})")
