"""Dump the SASS of the kernels whose mangled name contains PATTERN from the built library:
python scripts/sass_fn.py PATTERN [out]  (prints instruction / STL / LDL counts)."""
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2504_13339_b200" / "lib" / "libvegsplat_b200.so"


def main(pat, out=None):
    s = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    parts = s.split("Function : ")[1:]
    for p in parts:
        name = p.split("\n", 1)[0].strip()
        if pat in name:
            ins = [l for l in p.split("\n") if "/*" in l and ";" in l]
            print(name, "instructions", len(ins), "STL", sum("STL" in l for l in ins), "LDL",
                  sum("LDL" in l for l in ins))
            if out:
                Path(out).write_text(p)
            return


if __name__ == "__main__":
    main(*sys.argv[1:])
