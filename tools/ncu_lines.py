"""Per-source-line executed-instruction and stall-sample shares of one kernel in an ncu report."""
import collections, csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", k, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if 'Instructions Executed' in r)
ie, sa = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
cur = None; agg = collections.Counter(); st = collections.Counter(); src = {}; fname = ''
tot = tots = 0
for r in rows:
    if not r or r is h:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r[0] in ('Function Name', 'Line No'):
        continue
    if r[0].strip():
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        src[cur] = r[1].strip()[:100]; continue
    try:
        c, s = int(r[ie]), int(r[sa])
    except (ValueError, IndexError):
        continue
    agg[cur] += c; st[cur] += s; tot += c; tots += s
for key, c in agg.most_common(top):
    print(f"{c / tot * 100:5.1f}% st{st[key] / max(1, tots) * 100:5.1f}% {key[0][:10]}:{key[1]:4d} {src.get(key, '')}")
