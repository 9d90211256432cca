"""Instruction mix of the innermost loops of a cubin's SASS (development aid).

    python tools/sass_loops.py file.cubin [min_ffma2]
Lists every backward branch whose body holds >= min_ffma2 FFMA2 with its
size and top opcodes.
"""
import re
import subprocess
import sys
from collections import Counter

def main():
    path = sys.argv[1]
    need = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn = None
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if ins:
                report(fn, ins, need)
            fn, ins = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    if ins:
        report(fn, ins, need)

def report(fn, ins, need):
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, text) in enumerate(ins):
        m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d, )?0x([0-9a-f]+)", text)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        body = ins[addr[tgt]:i + 1]
        ops = Counter()
        for _, t in body:
            t = re.sub(r"^@!?U?P\w+\s+", "", t)
            ops[t.split()[0]] += 1
        if ops.get("FFMA2", 0) >= need:
            top = " ".join(f"{k}:{v}" for k, v in ops.most_common(12))
            print(f"{fn[:60]} loop {tgt:#x}-{a:#x} n={len(body)} {top}")

main()
