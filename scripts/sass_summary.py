"""Per-kernel SASS mnemonic counts of the built library (CPU; cuobjdump).

Evidence that the hot kernels use the Blackwell paths: UTCHMMA/UTCQMMA (tcgen05.mma),
UTMALDG (TMA tensor loads), UBLKCP (bulk copies), LDTM (tcgen05.ld from TMEM), HMMA
(mma.sync), SYNCS (mbarrier ops).

    python scripts/sass_summary.py > profiles/sass_summary_r02.txt
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

SO = Path(__file__).resolve().parents[1] / "paper_2602_00269_b200" / "libvoxb200.so"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "HMMA", "SYNCS",
        "ELECT", "FFMA", "MUFU"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else str(SO)
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    per = defaultdict(Counter)
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op.startswith(k):
                    per[cur][k] += 1
            per[cur]["_total"] += 1
    names = list(per)
    demangle = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS mnemonic counts per kernel in {Path(so).name} (sm_100a)")
    print("# kernel | instructions | " + " | ".join(KEYS))
    for name, dn in sorted(zip(names, demangle)):
        cnt = per[name]
        short = re.sub(r"\(.*", "", dn)[:80]
        print(f"{short} | {cnt['_total']} | " + " | ".join(str(cnt[k]) for k in KEYS))


if __name__ == "__main__":
    main()
