"""Summarise an ncu SASS source-page CSV: opcode histogram and hot basic blocks (dev tool).
    python tools/dev/sass_hot.py page.csv [dump_from dump_to]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
H = rows[1]
ie = H.index('Instructions Executed')
sm = H.index('Warp Stall Sampling (All Samples)')
te = H.index('Avg. Threads Executed')
body = [(r[1].strip(), int(r[ie] or 0), int(r[sm] or 0), r[te]) for r in rows[2:] if len(r) == len(H)]
if len(sys.argv) > 3:
    for i in range(int(sys.argv[2]), int(sys.argv[3])):
        ins, n, smp, t = body[i]
        if n:
            print(i, n, smp, t, ins[:95])
    sys.exit()
tot = sum(b[1] for b in body)
print('total', tot, 'n', len(body))
c, s = Counter(), Counter()
for ins, n, smp, _ in body:
    op = (ins.split()[1] if ins.startswith('@') else ins.split()[0]).split('.')[0]
    c[op] += n
    s[op] += smp
for op, n in c.most_common(24):
    print(f"{op:10s} {n:12d} {n / tot * 100:5.1f}% samples {s[op]}")
blocks, cur = [], None
for i, (ins, n, smp, t) in enumerate(body):
    if cur and cur[2] == n:
        cur[1] = i
        cur[3] += n
        cur[4] += smp
    else:
        cur = [i, i, n, n, smp]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
print('top blocks [start, end, count, total, samples] avg-threads')
for b in blocks[:20]:
    print(b, body[b[0]][3])
