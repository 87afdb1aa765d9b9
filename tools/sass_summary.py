"""Static SASS instruction counts per kernel of libhx.so (cuobjdump -sass) -> stdout.
usage: python tools/sass_summary.py [libhx.so] > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1805_08998_b200/libhx.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", out)),
                       capture_output=True, text=True).stdout.split("\n")
ops = ["DMMA", "LDGSTS", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG", "BAR", "SHFL", "DFMA"]
cnt = collections.OrderedDict()
cur = None
it = iter(names)
for line in out.split("\n"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = next(it).split("(")[0].replace("void ", "").replace("hx::", "")
        cnt[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        for o in ops:
            if op.startswith(o):
                cnt[cur][o] += 1
print("# round 2 (session 4): static SASS instruction counts per kernel of libhx.so (cuobjdump -sass, sm_100a)")
print("# DMMA = mma.sync.m8n8k4.f64 (FP64 tensor core; there is no tcgen05 kind::f64), LDGSTS = cp.async,")
print("# UBLKCP = cp.async.bulk (tried for the GEMM staging and measured slower: not in the shipped kernels),")
print("# SYNCS = mbarrier (try_wait / arrive), BAR = CTA / named barrier")
print(f"{'kernel':72s}" + "".join(f"{o:>8s}" for o in ops))
for k, c in cnt.items():
    if c["DMMA"] or "gemm" in k:
        print(f"{k[:72]:72s}" + "".join(f"{c[o]:8d}" for o in ops))
print("# kernels without DMMA (QR, Jacobi, ACA / Lanczos / range-finder iteration, assembly, gathers): "
      + str(sum(1 for c in cnt.values() if not c["DMMA"])))
