"""SASS of the scan kernel as a listing (not just opcode counts): tools/sass_listing.py > profiles/rNN_sass_k_scan_flowcache.txt
Instruction lines of k_scan_flowcache<5, SoaSource> from the built library (cuobjdump -sass), encodings stripped, with an
index of the instructions that only exist because the kernel is written for sm_100a."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1803_11449_b200", "libdhsa_b200.so")
FUN = "_ZN4dhsa16k_scan_flowcacheILi5ENS_9SoaSourceELb0EEEvT0_PjNS_9DevParamsE"
NOTABLE = [("UBLKCP", "cp.async.bulk global->shared: the packet stream is staged by the TMA engine"),
           ("SYNCS", "mbarrier arrive/expect_tx and try_wait: completion of the bulk copies"),
           (".256", "256-bit global load: one flow-cache set (8 ways x 4 B = one 32-byte sector) per lane"),
           ("REDG", "fire-and-forget atomic OR into the sketch"),
           ("MATCH.ANY", "warp aggregation of REDs that hit the same word"),
           ("VOTE", "miss compaction into the per-warp queue"),
           ("CCTL", "cache control")]
out = subprocess.run(["cuobjdump", "-sass", "-fun", FUN, LIB], capture_output=True, text=True).stdout
lines = []
for raw in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\*", raw)
    if m:
        lines.append((m.group(1), re.sub(r"\s+", " ", m.group(2)).strip()))
print(f"# SASS of k_scan_flowcache<5, SoaSource> (sm_100a), {len(lines)} instructions; cuobjdump -sass of {os.path.relpath(LIB, ROOT)}")
print("# index of the Blackwell-path instructions (address: instruction)")
for key, why in NOTABLE:
    hits = [(a, t) for a, t in lines if key in t]
    print(f"#   {key:10s} x{len(hits):<4d} {why}")
    for a, t in hits[:3]:
        print(f"#       {a}: {t}")
print("# no UTMALDG / UTC*MMA / LDTM: nothing on this path is a 2-D tile move or a contraction")
print()
for a, t in lines:
    print(f"{a}: {t}")
