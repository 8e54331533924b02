#!/usr/bin/env python
"""Backward-branch loops of a cuobjdump -sass listing with their instruction mix (the hot trip
of a kernel is the loop with the most FFMA2).  usage: sass_loops.py file.sass [top]"""
import collections, re, sys
ins = []
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
    tgt = None
    if m and m.group(1):
        tgt = int(m.group(1), 16)
    if tgt is not None and tgt < a and tgt in addr_idx:
        body = [t for _, t in ins[addr_idx[tgt]: i + 1]]
        mix = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
        loops.append((mix["FFMA2"], len(body), hex(tgt), hex(a), mix))
loops.sort(key=lambda x: -x[0])
for f, n, t, a, mix in loops[: int(sys.argv[2]) if len(sys.argv) > 2 else 3]:
    movs = mix["MOV"] + mix["IMAD"]
    print(f"loop {t}-{a}: {n} instr, FFMA2 {f}, MOV+IMAD {movs}, " + ", ".join(f"{k} {v}" for k, v in mix.most_common(12)))

# straight-line segments starting at a back-branch target, up to the first branch: the trip
seen = set()
segs = []
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt in addr_idx and tgt not in seen:
        seen.add(tgt)
        j = addr_idx[tgt]
        body = []
        while j < len(ins):
            body.append(ins[j][1])
            if "BRA" in ins[j][1] and j != addr_idx[tgt]:
                break
            j += 1
        mix = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
        segs.append((mix["FFMA2"], len(body), hex(tgt), mix))
segs.sort(key=lambda x: -x[0])
for f, n, t, mix in segs[:2]:
    print(f"segment {t}: {n} instr, FFMA2 {f}, MOV+IMAD.MOV {mix['MOV'] + mix['IMAD']}, " + ", ".join(f"{k} {v}" for k, v in mix.most_common(12)))
