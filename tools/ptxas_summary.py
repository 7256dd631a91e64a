"""Registers / spills per solver kernel instantiation from paper_2407_03272_b200/csrc/ptxas_log.txt."""
import os, re, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
log = open(os.path.join(ROOT, "paper_2407_03272_b200", "csrc", "ptxas_log.txt")).read().splitlines()
cur = None
for ln in log:
    m = re.search(r"Compiling entry function '(\w+)'", ln)
    if m:
        cur = m.group(1)
        continue
    if cur and "ajm_solve" in cur:
        m1 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m1:
            spill = (int(m1.group(1)), int(m1.group(2)))
        m2 = re.search(r"Used (\d+) registers", ln)
        if m2:
            dem = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
            dem = dem.replace("void ajm_solve_kernel", "").replace("(AjmPass)", "")
            print(f"{dem:45s} regs {m2.group(1)} spill st/ld {spill}")
            cur = None
