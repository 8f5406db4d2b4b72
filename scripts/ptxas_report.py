"""Registers / spills / stack of every kernel in one translation unit (ptxas -v), or a
diff-friendly table:  python scripts/ptxas_report.py paper_1811_11141_b200/csrc/k_fused.cu [regex]"""
import re
import subprocess
import sys

src = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "-Xcompiler", "-fPIC", "-I", "include", "-c", "-Xptxas", "-v", "-o", "/tmp/ptxas_report.o", src],
                     capture_output=True, text=True).stderr.splitlines()
cur = None
rows = {}
for line in out:
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {})["stack"], rows[cur]["spill_st"], rows[cur]["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
for name, r in sorted(rows.items()):
    if pat and not pat.search(name):
        continue
    if "regs" in r or r.get("spill_st"):
        print(f"{r.get('regs', '-'):>4} regs  stack {r.get('stack', 0):>4}  spill st/ld {r.get('spill_st', 0):>4}/{r.get('spill_ld', 0):<4} {name[:110]}")
