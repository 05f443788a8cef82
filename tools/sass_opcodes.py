"""Per-kernel SASS opcode summary of the built library objects (cuobjdump -sass), the evidence that
the hot kernels are Blackwell-native: UTCHMMA (tcgen05.mma), UTMALDG/UTMASTG (TMA), LDTM/STTM
(TMEM), UBLKCP (bulk copies), SYNCS (mbarriers). usage: python tools/sass_opcodes.py > profiles/r02/sass_opcodes.jsonl"""
import collections
import json
import re
import subprocess
from pathlib import Path

OBJ = Path(__file__).resolve().parents[1] / "paper_2506_06095_b200" / "_lib" / "obj"
KEEP = ("UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "UBLKCP", "SYNCS",
        "MUFU.EX2", "FFMA2", "FADD2", "FMUL2", "HMMA", "ELECT", "LDSM", "LDGSTS")

for obj in sorted(OBJ.glob("*.o")):
    txt = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    for fn in re.split(r"\n\s*Function : ", txt)[1:]:
        name = fn.split("\n", 1)[0].strip()
        ops = collections.Counter(m.group(1) for m in re.finditer(
            r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z][A-Za-z0-9_.]+)", fn))
        key = {k: v for k, v in sorted(ops.items()) if k.startswith(KEEP)}
        if not any(k.startswith(("UTC", "UTMA", "LDTM", "STTM", "UBLKCP")) for k in key):
            continue
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip() or name
        print(json.dumps({"object": obj.name, "kernel": dem, "instructions": sum(ops.values()), "blackwell_ops": key}))
