"""Static SASS instruction count per source line of the step kernel body
(the one-warp fp32 instantiation by default).  usage: sass_lines.py LO HI [name]"""
import re, subprocess, os, tempfile, collections, sys
lo, hi = int(sys.argv[1]), int(sys.argv[2])
name = sys.argv[3] if len(sys.argv) > 3 else "step_kernelIftLi1ELi2ELi16ELb0E"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_1504_05158_b200/libqsb.so")], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
on = False; cur = None; addrs = []; last_exit = None; first_ret = None
for line in txt.split("\n"):
    if line.startswith(".text."): on = name in line; continue
    if not on: continue
    m = re.search(r'## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", line)
    if m:
        addrs.append(cur)
        if "RET.REL" in line and first_ret is None: first_ret = len(addrs)
        if "EXIT" in line and first_ret is None: last_exit = len(addrs)
src = open("paper_1504_05158_b200/csrc/step_kernel.cuh").read().split("\n")
c = collections.Counter(a[1] for a in addrs[:last_exit] if a and a[0] == "step_kernel.cuh" and lo <= a[1] <= hi)
for l, v in sorted(c.items()): print(f"{v:4d} {l:5d} {src[l-1].strip()[:100]}")
print("total", sum(c.values()))
