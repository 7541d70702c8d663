"""Static SASS size of a step_kernel instantiation, split into the kernel
body (step_kernel.cuh lines from the kernel's definition on, plus inlined
helpers called from it) and the out-of-line callees.  Usage:
sass_size.py [mangled-name-substring]"""
import re, subprocess, sys, collections, tempfile, os
name = sys.argv[1] if len(sys.argv) > 1 else "step_kernelIftLi1ELi2ELi16ELb0E"
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1504_05158_b200/libqsb.so"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
on = False; cur = None; addrs = []
for line in txt.split("\n"):
    if line.startswith(".text."):
        on = name in line; continue
    if not on: continue
    m = re.search(r'## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m:
        addrs.append((int(m.group(1), 16), cur))
        if "RET.REL" in line and "first_ret" not in globals(): first_ret = len(addrs)
        if "EXIT" in line and "first_ret" not in globals(): last_exit = len(addrs)
# the kernel body ends at the first RET-delimited callee: find the first
# instruction attributed to a step_kernel.cuh line below the kernel start
src = open("paper_1504_05158_b200/csrc/step_kernel.cuh").read().split("\n")
kline = next(i + 1 for i, l in enumerate(src) if l.startswith("step_kernel(const"))
body_end = None
for a, c in addrs:
    if a > 256 and c and c[0] == "step_kernel.cuh" and c[1] < kline - 60 and body_end is None:
        pass
tot = len(addrs)
by = collections.Counter()
for a, c in addrs:
    by[(c[0] if c else "?")] += 1
print(f"{name}: {tot} instrs = {tot*16/1024:.1f} KB")
first_callee = last_exit
print(f"kernel body (to its last EXIT): {first_callee} instrs = {first_callee*16/1024:.1f} KB")
ranges = []
marks = [("prologue", "step_kernel(const"), ("setup", "// ---- per-column registers"),
         ("velocity", "// ================= phase 1: velocity"), ("stats", "// ================= normalisation"),
         ("agg:init+endgame", "// ================= phase 2: aggregation"), ("agg:bulk", "// ---- bulk step"),
         ("agg:round/ties", "if (!bulk) {"), ("agg:retire", "// ---- retire row"),
         ("agg:rescans", "// ---- cooperative rescans"), ("agg:end", "// the tile is no longer read"),
         ("goal", "// ================= phase 3: goal"), ("pbest", "// ================= phase 4a")]
starts = []
for nm, mk in marks:
    i = next(i + 1 for i, l in enumerate(src) if mk in l and i + 1 >= kline - 1)
    starts.append((i, nm))
def region(l):
    r = "?"
    for s, nm in starts:
        if l >= s: r = nm
    return r
g = collections.Counter()
for a, c in addrs[:first_callee]:
    if c is None: g["?"] += 1
    elif c[0] == "step_kernel.cuh" and c[1] >= kline: g[region(c[1])] += 1
    else: g[c[0] if c[0] != "step_kernel.cuh" else "helpers"] += 1
for k, v in g.most_common(): print(f"  {v:5d} {k}")
