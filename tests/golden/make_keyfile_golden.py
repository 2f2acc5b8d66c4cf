"""Generate tests/golden/keyfiles/ from the REFERENCE ITSELF.

The reference's dataio (dataio.cpp: key-file writers and the mergebench
input generator), compiled unmodified into oracle/_ref/libmergepath_ref.so,
writes the files; tests/test_keyfile.py checks that the B200 side's
mp_keyfile_* and `mergebench_b200 gen` produce the same bytes and read them
back.  Small sizes: the files are committed.

    python tests/golden/make_keyfile_golden.py     # needs /root/reference
"""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import bindings  # noqa: E402

OUT = Path(__file__).resolve().parent / "keyfiles"
CASES = [  # (dist, na, nb, seed)
    ("uniform", 300, 200, 1), ("uniform", 0, 17, 5), ("uniform", 1000, 1000, 42),
    ("all_equal", 50, 30, 1), ("disjoint_ranges", 257, 129, 9),
    ("interleaved", 100, 99, 1),
]


def main() -> None:
    bindings.build()  # also builds oracle/_ref/ref_keyfile_gen
    gen = ROOT / "oracle" / "_ref" / "ref_keyfile_gen"
    OUT.mkdir(exist_ok=True)
    index = []
    for dist, na, nb, seed in CASES:
        stem = f"gen_{dist}_{na}_{nb}_{seed}"
        for fmt in ("bin", "text"):
            subprocess.run([str(gen), "gen", dist, str(na), str(nb), str(seed),
                            str(OUT / f"{stem}_a.{fmt}"), str(OUT / f"{stem}_b.{fmt}"), fmt],
                           check=True)
        index.append({"dist": dist, "na": na, "nb": nb, "seed": seed})
    (OUT / "index.json").write_text(json.dumps(index, indent=1) + "\n")
    print(f"wrote {len(index)} cases to {OUT}")


if __name__ == "__main__":
    main()
