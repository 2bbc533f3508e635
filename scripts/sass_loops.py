"""Experiment support: instruction mix of the loops of one kernel's SASS.

    cuobjdump -sass lib.so > x.sass; python scripts/sass_loops.py x.sass <kernel-substring>
Prints, for every backward branch (loop), its length and opcode histogram."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1]).read().split("\n")
key = sys.argv[2]
funcs, cur = {}, None
for ln in txt:
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            funcs[cur].append((int(m.group(1), 16), m.group(2)))
for name, ins in funcs.items():
    if key not in name:
        continue
    print("==", name, len(ins), "instructions")
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, op) in enumerate(ins):
        m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", op)
        m2 = re.search(r"BRA\s+`?\(?\.?L?_?x?_?\d*\)?\s*0x([0-9a-f]+)|BRA 0x([0-9a-f]+)", op)
        tgt = None
        mm = re.search(r"0x([0-9a-f]+)", op) if "BRA" in op else None
        if mm:
            tgt = int(mm.group(1), 16)
        if tgt is not None and tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            c = Counter(re.sub(r"^@!?U?P\w+\s+", "", o).split()[0].split(".")[0] for _, o in body)
            if len(body) > 40:
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr:", ", ".join(f"{k}={v}" for k, v in c.most_common(14)))
