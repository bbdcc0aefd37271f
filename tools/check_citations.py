"""Check every `src/<module>.py:<line>[-<line>]` citation in the repo against
the reference file's length (build container only: reads /root/reference)."""
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/pkg/src/permanent")
pat = re.compile(r"(?:src/|permanent/)?(\b[a-z_]+\.py):((?:\d+(?:-\d+)?)(?:,\s*\d+(?:-\d+)?)*)")
bad = 0
for p in ROOT.rglob("*"):
    if p.suffix not in (".py", ".cu", ".cuh", ".h", ".md", ".c") or "scratch_reftests" in p.parts:
        continue
    if p.name in ("SURVEY.md", "VERDICT.md", "ADVICE.md", "BASELINE.md"):
        continue
    for no, line in enumerate(p.read_text(errors="ignore").splitlines(), 1):
        for mod, spans in pat.findall(line):
            ref = SRC / mod
            if not ref.exists():
                continue
            n = len(ref.read_text().splitlines())
            for span in re.split(r",\s*", spans):
                hi = int(span.split("-")[-1])
                if hi > n:
                    bad += 1
                    print(f"{p.relative_to(ROOT)}:{no}: {mod}:{span} beyond {n} lines")
sys.exit(1 if bad else 0)
