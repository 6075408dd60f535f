"""Build a tuning variant of the library: one translation unit recompiled with extra -D
flags, linked with the other (already built) objects into _lib/libpcfb200.<name>.so;
load it with PCF_LIB_VARIANT=<name>.

    python tools/build_variant.py NAME SOURCE.cu -DFOO=1 [-DBAR=2 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
g.build_lib()
objdir = os.path.join(g.PKG, "_lib", "obj")
flags = [f for f in g.NVCC_FLAGS if f not in ("-shared", "-ldl")]
vobj = os.path.join("/tmp", f"{name}_{os.path.basename(src)}.o")
subprocess.run([g._nvcc(), *flags, *defs, "-c", "-o", vobj, os.path.join(g.CSRC, src)],
               check=True, cwd=g.CSRC)
objs = [vobj if o == os.path.basename(src).lstrip("_").replace("old_", "pcf_") + ".o" else os.path.join(objdir, o)
        for o in sorted(os.listdir(objdir)) if o.endswith(".o")]
out = os.path.join(g.PKG, "_lib", f"libpcfb200.{name}.so")
subprocess.run([g._nvcc(), *g.NVCC_FLAGS, "-o", out, *objs], check=True, cwd=g.CSRC)
print(out)
