"""Opcode mix of one kernel from `ncu -i REP --page source --csv --print-source sass` output.
usage: python tools/sass_mix.py SASS.csv POINTS"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
npt = float(sys.argv[2])
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
hdr = rows[hi]
ix, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
iw, ist = hdr.index("L1 Wavefronts Shared"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, wf, st = collections.Counter(), collections.Counter(), collections.Counter()
tot = tst = 0
for r in rows[hi + 1:]:
    if len(r) <= ix or not r[ix].strip().isdigit():
        continue
    toks = r[isrc].strip().split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
    n = int(r[ix] or 0)
    cnt[op] += n; tot += n; wf[op] += int(r[iw] or 0); st[op] += int(r[ist] or 0); tst += int(r[ist] or 0)
print("total warp instr/pt %.2f  smem wavefronts/pt %.2f" % (tot / npt, sum(wf.values()) / npt))
for op, n in cnt.most_common(26):
    print("%-10s %6.3f /pt  %5.1f%%  wf/pt %.3f  stall %.1f%%" % (op, n / npt, 100 * n / tot, wf[op] / npt, 100 * st[op] / max(tst, 1)))
