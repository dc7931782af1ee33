"""Build a scratch libsse.so whose K6 v4 stage loop is instantiated per one-/two-tile warp
(the experiment that hung); output under /tmp/k6h (never the in-tree build)."""
import os, shutil, subprocess, sys
src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "paper_1912_08810_b200", "csrc")
dst = "/tmp/k6h/pkg/csrc"  # sse_capi.cu includes ../../include/sse.h
os.makedirs(dst, exist_ok=True)
shutil.copytree(os.path.join(src, "..", "..", "include"), "/tmp/k6h/include", dirs_exist_ok=True)
for f in ("sse_capi.cu", "sse_kernels.cuh"):
    shutil.copy(os.path.join(src, f), dst)
s = open(os.path.join(src, "sse_kernels.cu")).read()
old_start = "  for (int ss = 0; ss < n_ss; ++ss) {\n    const int slot = ss % SL;\n    const int st = ss / kPi3Sub, j = ss - st * kPi3Sub;\n    const int kq = j * QS;\n"
i = s.index(old_start, s.index("pi_dmma4_kernel(PiArgs p"))
j = s.index("\n  if (!active) return;\n  double2* part = p.partial + ((((long long)la * 2 + pol)", i)
body = s[i:j].replace("if (live && two) {", "if (live && TWO) {")
new = ("  auto run = [&](auto two_c) {\n    constexpr bool TWO = decltype(two_c)::value;\n" + body + "\n  };\n"
       "  if (two) run(std::true_type{});\n  else run(std::false_type{});\n")
s = s[:i] + new + s[j:]
s = s.replace("#include <cstdlib>", "#include <cstdlib>\n#include <type_traits>")
if os.environ.get("K6_SYNCWARP"):  # lane 0 releases the slot only after the whole warp is done with it
    k = s.index("pi_dmma4_kernel(PiArgs p")
    a = s.index("    if (lane == 0) mbar_arrive(empty + slot);\n", k)
    s = s[:a] + "    __syncwarp();\n" + s[a:]
open(os.path.join(dst, "sse_kernels.cu"), "w").write(s)
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
       "-shared", "-o", "/tmp/k6h/libsse.so", os.path.join(dst, "sse_kernels.cu"), os.path.join(dst, "sse_capi.cu"),
       "-I", os.path.join(src, "..", "..", "include")]
r = subprocess.run(cmd, capture_output=True, text=True)
print(r.returncode, r.stderr[-2000:])
sys.exit(r.returncode)
