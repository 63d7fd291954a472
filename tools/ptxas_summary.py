"""Summarise nvcc -Xptxas -v logs in build/ublr: kernel, registers, spills, smem."""
import glob, re, subprocess, sys
for f in sorted(glob.glob("build/ublr/*.ptxas.txt")):
    cur = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            try:
                name = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
            except Exception:
                pass
            name = re.sub(r"ublr::\(anonymous namespace\)::", "", name)
            cur = [name[:90], "", "", ""]
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            cur[2] = f"spill {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line)
        if m and cur:
            cur[1] = f"regs {m.group(1)}"
            cur[3] = f"smem {m.group(2)}"
            print(f"{cur[0]:90s} {cur[1]:9s} {cur[2]:14s} {cur[3]}")
            cur = None
