"""Write tests/golden/base_hashes.txt: SHA-256 of each BASELINE config's base matrix.

Calls only the seeded input generator (inputs/), never the CUDA path.  The
hash freezes the constructor: any change to it must
regenerate this file in the same commit and say why.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import inputs  # noqa: E402

if __name__ == "__main__":
    out = ROOT / "tests" / "golden" / "base_hashes.txt"
    lines = ["# config  sha256(shape|Z|base int16 LE)  -- written by tools/write_goldens.py"]
    for name in ("C1", "C2", "C3a", "C3b", "C4", "T24", "P2048", "P8192"):   # P*: QC-PEG (inputs/peg.py)
        base, Z = inputs.config_base(name)
        lines.append(f"{name} {inputs.base_sha256(base, Z)}")
    out.write_text("\n".join(lines) + "\n")
    print(out.read_text())
