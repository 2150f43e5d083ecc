"""List the loops of a SASS dump (backward branches): body length, LDG / RED / ATOM counts.

usage: python tools/sass_loops.py file.sass   (output of cuobjdump -sass for one function)
"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr:
            body = [x for _, x in ins[addr[tgt]:i + 1]]
            n = len(body)
            cnt = lambda k: sum(1 for x in body if re.search(k, x))
            print(f"loop {tgt:#06x}-{a:#06x}: {n} instr, LDG {cnt('LDG')}, RED {cnt('RED')}, "
                  f"I2F {cnt('I2F')}, IMAD.WIDE {cnt('IMAD.WIDE')}, ISETP {cnt('ISETP')}")
