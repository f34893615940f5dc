"""List backward-branch loops of a SASS dump with their instruction mix."""
import re, sys
from collections import Counter
ins = []
for l in open(sys.argv[1]):
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
def op(s):
    t = s.split()
    if t[0].startswith('@'):
        t = t[1:]
    return t[0]
minf = int(sys.argv[2]) if len(sys.argv) > 2 else 32
for i, (a, s) in enumerate(ins):
    if 'BRA' in s:
        m = re.search(r'BRA[^0-9]*0x([0-9a-f]+)', s)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr:
                body = [x for _, x in ins[addr[tgt]:i + 1]]
                c = Counter(op(x).split('.')[0] for x in body)
                if c['FFMA'] + c['DFMA'] >= minf:
                    print(f"loop {tgt:x}-{a:x} len={len(body)} FFMA={c['FFMA']} DFMA={c['DFMA']} LDS={c['LDS']} LD={c['LD']} "
                          + str({k: v for k, v in c.most_common(12) if k not in ('FFMA', 'LDS', 'LD', 'DFMA')}))
