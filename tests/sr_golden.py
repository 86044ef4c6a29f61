"""SR codec fixtures from the reference itself, usable without /root/reference:

* REF_TEST_WIRE: the golden bytes of the reference's own test "wire format golden bytes"
  (proj/tests/test_sparsecomp.cpp:258-279): h=1, m=2, shared = 0, expert w_up = {0.5,
  -1.25}, w_down = {0, 2}, k = 2 -> entries (1, -1.25f), (3, 2.0f).
* cases(): tests/golden/sr_cases.npz, written by oracle/gen_golden.py from the
  UNMODIFIED reference library (oracle/_ref): seeded demo experts (continuous and
  heavy-tie), joint and per-matrix budgets, 32/64-bit widths, k = 0 and k >= P, with the
  reference's wire bytes and decoded experts.
"""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

REF_TEST_EXPERT = np.array([0.5, -1.25, 0.0, 2.0], np.float32)
REF_TEST_SHARED = np.zeros(4, np.float32)
REF_TEST_WIRE = bytes([ord("S"), ord("R"), ord("C"), ord("1"),
                       0x01, 0x00, 0x00, 0x00,
                       0x02, 0x00, 0x00, 0x00,
                       0x02, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00,
                       0x20, 0x00, 0x00, 0x00,
                       0x20, 0x00, 0x00, 0x00,
                       0x01, 0x00, 0x00, 0x00, 0x00, 0x00, 0xa0, 0xbf,
                       0x03, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0x40])


def cases():
    """[(name, dict(h, m, ratio, k, iw, vw, per_matrix, expert, shared, wire, decoded))]"""
    d = np.load(os.path.join(GOLDEN, "sr_cases.npz"))
    out = []
    i = 0
    while f"c{i}_spec" in d.files:
        h, m, ratio, k, iw, vw, pm = d[f"c{i}_spec"].tolist()
        out.append((f"c{i}", dict(h=int(h), m=int(m), ratio=None if ratio < 0 else ratio,
                                  k=None if k < 0 else int(k), iw=int(iw), vw=int(vw), per_matrix=bool(pm),
                                  expert=d[f"c{i}_expert"], shared=d[f"c{i}_shared"], wire=d[f"c{i}_wire"],
                                  decoded=d[f"c{i}_decoded"])))
        i += 1
    return out
