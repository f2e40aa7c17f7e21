"""Executed-instruction mix of a kernel from an ncu capture's SASS source
page: thread instructions per opcode class, per path.

    python tools/sass_mix.py <rep.ncu-rep> <paths per launch> [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, paths = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ti, wi = hdr.index("Source"), hdr.index("Thread Instructions Executed"), \
    hdr.index("Instructions Executed")
ops = Counter()
warp = Counter()
for r in rows[2:]:
    if len(r) <= ti:
        continue
    src = r[si].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    op = m.group(2)
    ops[op] += float(r[ti] or 0)
    warp[op] += float(r[wi] or 0)
CLS = {"fp32": {"FFMA", "FMUL", "FADD", "FMNMX", "FSWZADD", "FMUL2", "FFMA2", "FADD2"},
       "mufu": {"MUFU"},
       "int": {"IMAD", "IADD3", "IADD", "LOP3", "SHF", "IMNMX", "LEA", "IABS", "POPC", "FLO",
               "BREV", "IMUL", "VIMNMX", "IADD32I", "LOP32I", "SGXT", "IMAD_WIDE"},
       "cmp/sel": {"FSETP", "ISETP", "FSEL", "SEL", "PLOP3", "P2R", "R2P", "FCHK", "DSETP"},
       "conv": {"F2I", "I2F", "F2F", "I2FP", "F2IP", "FRND"},
       "mem": {"LDS", "STS", "LDG", "STG", "LD", "ST", "LDC", "ULDC", "RED", "ATOM", "LDL", "STL",
               "ATOMS"},
       "ctrl": {"BRA", "BSSY", "BSYNC", "WARPSYNC", "EXIT", "CALL", "RET", "BMOV", "NOP", "YIELD",
                "VOTE", "VOTEU", "SHFL", "MATCH", "REDUX", "BREAK", "JMP", "S2R", "CS2R", "S2UR",
                "UMOV", "UIADD3", "ULOP3", "USHF", "UISETP", "USEL", "ELECT", "BPT", "UFLO",
                "UPOPC", "R2UR", "UMOV", "ULEA"},
       "mov": {"MOV", "PRMT", "MOVM"}}
cls = Counter()
for op, v in ops.items():
    c = next((k for k, s in CLS.items() if op in s), "other:" + op)
    cls[c] += v
tot = sum(ops.values())
print(f"thread instructions per path: {tot / paths:.1f}  (warp instr {sum(warp.values()):.3e})")
for c, v in cls.most_common():
    print(f"  {c:14s} {v / paths:8.1f}  {v / tot:6.1%}")
print("top opcodes:")
for op, v in ops.most_common(top):
    print(f"  {op:10s} {v / paths:8.1f}  {v / tot:6.1%}  lanes {v / max(warp[op], 1):.1f}")
