"""Raw-binary KAT for tests/c/abi_kat.c, derived from the committed reference goldens
(scheme_default.npz: n01 = hom_nand(ct0, ct1) as the reference computed it; both fresh, so no
swap).  Layout: u32 header (n, ell, q, m, words) then ct0, ct1, n01 as dense u32 rows."""
import os
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
z = np.load(os.path.join(HERE, "scheme_default.npz"))
n, q, m, ell = 8, (1 << 29) - 3, 32, 29
words = z["ct0"].size
hdr = np.array([n, ell, q, m, words], dtype="<u4")
blob = np.concatenate([hdr] + [np.ascontiguousarray(z[k], dtype="<u4").ravel() for k in ("ct0", "ct1", "n01")])
blob.tofile(os.path.join(HERE, "kat_default_nand.bin"))
print(len(blob) * 4, "bytes")
