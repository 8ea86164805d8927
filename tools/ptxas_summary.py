"""Per-kernel registers / spills from a verbose build (nvcc -Xptxas -v)."""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, "paper_2112_06465_b200/_build.py", "--force", "-v"],
                     capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_\w+?)(E|I)", name)
        cur = k.group(1) if k else name[:40]
        if "ILi0E" in name:
            cur += "<0>"
        if "ILi1E" in name:
            cur += "<1>"
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:28s} regs={m.group(1):>4s} spill_st/ld={spill}")
        cur = None
