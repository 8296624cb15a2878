"""Regenerate profiles/<tag>_sass_evidence.txt and <tag>_ptxas.txt from the
built libsg.so / sources (run in the build container):

    python tools/sass_evidence.py r02

SASS: per kernel the opcodes that prove the memory-path design -- TMA bulk
copies (UBLKCP), mbarrier operations (SYNCS.*), shared / global atomics,
warp votes and matches -- and that no tensor-core op is issued (these are
integer gather/scatter kernels).  ptxas: registers, spills, barriers and
static shared memory per kernel."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1002_4482_b200 import build  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
lib = build.LIB
ops = ("UBLKCP", "UTMALDG", "SYNCS", "ATOMS", "ATOMG", "RED", "VOTE", "MATCH", "REDUX", "HMMA", "UTCMMA", "UTCQMMA")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
demangled = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
out = [f"SASS evidence for libsg.so (cuobjdump -sass paper_1002_4482_b200/libsg.so, sm_100a), {tag}",
       "Per kernel: TMA bulk copies (UBLKCP), mbarrier ops (SYNCS.*), shared/global atomics, votes, matches, "
       "tensor-core ops (none expected).", ""]
cur, cnt = None, collections.Counter()


def flush():
    if cur:
        out.append(cur[:110])
        out.append("    " + str(dict(sorted(cnt.items()))))


for line in demangled.splitlines():
    m = re.match(r"\s*Function : (.*)", line)
    if m:
        flush()
        cur, cnt = m.group(1).replace("sg::", ""), collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(2)
        for o in ops:
            if op == o or op.startswith(o):
                cnt[o] += 1
flush()
open(os.path.join(ROOT, "profiles", f"{tag}_sass_evidence.txt"), "w").write("\n".join(out) + "\n")

lines = [f"ptxas -v (nvcc, {' '.join(build.ARCH)} -O3): registers, spills and static smem per kernel of libsg, {tag}", ""]
for src in build.SOURCES:
    if not src.endswith(".cu"):
        continue
    r = subprocess.run(["nvcc", *build.ARCH, "-O3", "-std=c++17", "-I", build.INCLUDE, "-Xptxas", "-v", "-c",
                        os.path.join(build.CSRC, src), "-o", "/dev/null"], capture_output=True, text=True)
    fn = None
    for l in r.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\w+)'", l)
        if m:
            fn = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            fn = fn.replace("sg::", "").split("(")[0]
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", l)
        if m and fn:
            stack = m.groups()
        m = re.search(r"Used (\d+) registers(.*)", l)
        if m and fn:
            lines.append(f"{fn[:80]:80s} regs {int(m.group(1)):3d}  stack {stack[0]} B, spill st/ld {stack[1]}/{stack[2]} B "
                         f"{m.group(2).strip(', ')}")
            fn = None
open(os.path.join(ROOT, "profiles", f"{tag}_ptxas.txt"), "w").write("\n".join(lines) + "\n")
print("ok")
