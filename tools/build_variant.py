"""Build a variant of libddm.so with extra nvcc -D flags (dev A/B timing).
usage: build_variant.py NAME [--rev GITREV] [-DFLAG=V ...]  ->  variants/libddm_NAME.so
(load with DDM_LIB=...); --rev builds the csrc/ of a git revision instead of the work tree."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06680_b200 import _build as B
name, defs = sys.argv[1], sys.argv[2:]
csrc = B.CSRC
if defs[:1] == ["--rev"]:
    rev, defs = defs[1], defs[2:]
    import tempfile
    top = tempfile.mkdtemp(prefix="ddmrev_")
    csrc = os.path.join(top, "pkg", "csrc")
    os.makedirs(csrc)
    os.makedirs(os.path.join(top, "include"))
    blob = subprocess.run(["git", "-C", B.ROOT, "show", f"{rev}:include/ddm.h"], capture_output=True, check=True).stdout
    open(os.path.join(top, "include", "ddm.h"), "wb").write(blob)
    for f in B.SOURCES + B.HEADERS:
        blob = subprocess.run(["git", "-C", B.ROOT, "show", f"{rev}:paper_1703_06680_b200/csrc/{f}"],
                              capture_output=True, check=True).stdout
        open(os.path.join(csrc, f), "wb").write(blob)
out = os.path.join(B.ROOT, "variants", f"libddm_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [B.nvcc(), *B.NVCC_FLAGS, *defs, "-I", os.path.join(B.ROOT, "include"), "-o", out,
       *[os.path.join(csrc, f) for f in B.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-4000:])
print("built", out)
