"""Generate the SFAB / manifest fixtures with the REAL reference ``factorfit.data_io``.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_sfab.py

Writes ``tests/golden/sfab/``: a manifest of three small subjects (one with
coordinates) written by the reference's ``save_matrix`` / ``write_manifest``,
plus ``malformed/*.sfab`` containers together with the exception the
reference raises for each (``expected.json``: class, field, offset).  The
tests compare the native reader/writer against these files; nothing at
test time reads /root/reference.
"""

import json
import shutil
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "sfab"


def main():
    sys.path.insert(0, str(REF_SRC))
    from factorfit import data_io  # noqa: E402

    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "subjects").mkdir(parents=True)
    (OUT / "malformed").mkdir()
    rng = np.random.default_rng(20261020)
    entries = []
    for i, v in enumerate((37, 52, 41)):
        x = rng.standard_normal((v, 12))
        p = OUT / "subjects" / f"sub-{i:02d}.sfab"
        data_io.save_matrix(p, x)
        coords = None
        if i == 1:
            coords = OUT / "subjects" / f"sub-{i:02d}_coords.sfab"
            data_io.save_matrix(coords, rng.integers(0, 9, size=(v, 3)).astype(np.float64))
        entries.append(data_io.ManifestEntry(f"sub-{i:02d}", p, coords))
    man = data_io.Manifest("golden", entries, (9, 9, 9))
    data_io.write_manifest(OUT / "manifest.json", man)

    good = (OUT / "subjects" / "sub-00.sfab").read_bytes()
    cases = {
        "bad_magic": b"SFAX" + good[4:],
        "bad_version": good[:4] + (2).to_bytes(4, "little") + good[8:],
        "bad_dtype": good[:8] + (1).to_bytes(4, "little") + good[12:],
        "short_header": good[:20],
        "short_payload": good[:-8],
        "trailing": good + b"\x00",
    }
    expected = {}
    for name, blob in cases.items():
        p = OUT / "malformed" / f"{name}.sfab"
        p.write_bytes(blob)
        try:
            data_io.load_matrix(p)
            expected[name] = None
        except Exception as e:  # noqa: BLE001
            expected[name] = {"class": type(e).__name__, "field": getattr(e, "field", None),
                              "offset": getattr(e, "offset", None)}
    (OUT / "malformed" / "expected.json").write_text(json.dumps(expected, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
