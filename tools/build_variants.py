"""Build tuning variants of the library under build/variants/ for A/B runs (tools/gpu_ab.sh):
python tools/build_variants.py name1:DEF1=V,DEF2=V name2:..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_11449_b200 import _build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    out = os.path.join("build", "variants", f"{name}.so")
    import subprocess
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, "-Xptxas", "-v", *[f"-D{d}" for d in defs.split(",") if d], "-o", out,
           *[os.path.join(_build.CSRC, f) for f in _build.SOURCES]]
    os.makedirs(os.path.dirname(out), exist_ok=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode:
        print(proc.stderr[-3000:])
        sys.exit(1)
    lines = proc.stderr.splitlines()
    for i, l in enumerate(lines):
        if "k_scan_flowcacheILi5ENS_9SoaSource" in l and "Compiling" in l:
            print(name, "|", lines[i + 2].strip(), "|", lines[i + 3].strip())
