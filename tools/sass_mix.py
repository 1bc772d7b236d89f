"""Static opcode mix of the plan-specialised kernel's hot loop (design check without a GPU):
   python tools/sass_mix.py build/jit_C5.cubin
The hot loop is taken as the largest backward-branch range in gace_jit_probe."""
import collections
import re
import subprocess
import sys

sass = subprocess.run(["cuobjdump", "-sass", "-fun", "gace_jit_probe", sys.argv[1]], capture_output=True, text=True).stdout
ins = []
for line in sass.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = (0, 0)
for addr, txt in ins:
    m = re.search(r"BRA\s+(?:\w+,\s*)?(0x[0-9a-f]+)", txt)
    if m and "BRA" in txt.split()[0 if not txt.startswith("@") else 1]:
        tgt = int(m.group(1), 16)
        if tgt < addr and addr - tgt > best[1] - best[0]:
            best = (tgt, addr)
ALU = {"LOP3", "SHF", "ISETP", "LEA", "IADD3", "SEL", "VIMNMX", "VIMNMX3", "FLO", "PRMT", "IABS", "VIADD", "VIADDMNMX", "P2R", "R2P", "PLOP3"}
FMA = {"IMAD", "IMAD.HI", "IMAD.WIDE", "IMAD.SHL", "IMAD.MOV", "IMAD.IADD", "IMAD.X", "IMAD.U32"}
c = collections.Counter()
for addr, txt in ins:
    if best[0] <= addr <= best[1]:
        t = txt.split()
        op = t[1] if t[0].startswith("@") else t[0]
        c[op.split(".")[0] if not op.startswith("IMAD") else "IMAD"] += 1
alu = sum(n for o, n in c.items() if o in ALU)
fma = c["IMAD"]
print(f"hot loop {best[0]:#x}-{best[1]:#x}: {sum(c.values())} instructions, ALU-pipe {alu}, FMA-pipe {fma}")
print("  " + "  ".join(f"{o} {n}" for o, n in c.most_common(30)))
