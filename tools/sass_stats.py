#!/usr/bin/env python
"""Per-loop SASS opcode statistics for a cubin / .so (cuobjdump -sass).

For every kernel, finds backward branches (loops), and prints the opcode mix
of each loop body: the evidence for "LOP3 per keystream clock" and for where
spills (LDL/STL) sit.  Usage: tools/sass_stats.py <file> [kernel-substring]
"""
import collections
import re
import subprocess
import sys


def main():
    path = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    txt = subprocess.run(["cuobjdump", "-sass", path], stdout=subprocess.PIPE, text=True, check=True).stdout
    kernels = re.split(r"\n\s*Function : ", txt)[1:]
    ins_re = re.compile(r"^\s+/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)\s*(.*?);")
    for k in kernels:
        name = k.split("\n", 1)[0].strip()
        if filt not in name:
            continue
        ins = []
        for line in k.splitlines():
            m = ins_re.match(line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2), m.group(3)))
        total = collections.Counter(op.split(".")[0] for _, op, _ in ins)
        print(f"== {name}: {len(ins)} instructions")
        print("   total:", dict(total.most_common(12)))
        for addr, op, args in ins:
            if op.startswith("BRA"):
                m = re.search(r"0x([0-9a-f]+)", args)
                if m and int(m.group(1), 16) < addr:
                    lo = int(m.group(1), 16)
                    body = [o for a, o, _ in ins if lo <= a <= addr]
                    c = collections.Counter(o.split(".")[0] for o in body)
                    alu = sum(v for o, v in c.items() if o in ("LOP3", "IADD3", "SHF", "PRMT", "LEA", "ISETP", "SEL", "IADD", "LOP", "SGXT", "BMSK", "VIADD", "IABS", "IMNMX", "VIMNMX", "FMNMX"))
                    print(f"   loop 0x{lo:x}..0x{addr:x}: {len(body)} instr, ALU-pipe {alu}: {dict(c.most_common(14))}")


if __name__ == "__main__":
    main()
