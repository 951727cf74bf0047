"""Registers / stack (spill) per rollout variant from cuobjdump --dump-resource-usage."""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "--dump-resource-usage", sys.argv[1] if len(sys.argv) > 1 else
                      "paper_2001_04931_b200/libempc_b200.so"], capture_output=True, text=True).stdout
fn = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1); continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and fn:
        k = re.search(r"rollout_kernelI([fd])[a-z]*Li(\d+)ELi(\d+)ELi(\d+)ELb([01])ELb([01])ELi(\d+)ELi(\d+)", fn)
        if k:
            print(f"{k.group(1)} NP={k.group(2)} RR={k.group(3)} CC={k.group(4)} areg={k.group(5)} dq={k.group(6)} ks={k.group(7)} maxt={k.group(8)} REG={m.group(1)} STACK={m.group(2)}")
        elif "select" in fn or "finalize" in fn:
            print(fn[:40], "REG", m.group(1), "STACK", m.group(2))
        fn = None
