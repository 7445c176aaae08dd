# quick diagnostic: TC kernel vs oracle with both descriptor variants
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import gsw
from paper_1611_08769_b200 import GswScheme, DEFAULT_PARAMS, EXACT_PARAMS
for params, op in ((EXACT_PARAMS, gsw.EXACT), (DEFAULT_PARAMS, gsw.DEFAULT)):
    s = GswScheme(params)
    rng = np.random.default_rng(0)
    a = rng.integers(0, params.q, (4, params.n_ct, params.k)).astype(np.uint32)
    b = rng.integers(0, params.q, (4, params.n_ct, params.k)).astype(np.uint32)
    want = [gsw.hom_nand_compact(op, a[i], b[i]) for i in range(4)]
    for kern in (1, 2):
        for dbg in ((0, 1) if kern == 1 else (0, 2, 4)):
            s.ctx.set_kernel(kern); s.ctx.set_debug(dbg)
            try:
                got = s.ctx.nand_batch(a, b).astype(np.int64)
                ok = all(np.array_equal(got[i], want[i]) for i in range(4))
                rows_bad = sorted(set(np.nonzero((got[0] != want[0]).any(axis=1))[0].tolist()))
                print(params.n, 'kernel', kern, 'dbg', dbg, 'OK' if ok else f'MISMATCH rows {rows_bad[:10]}.. n={len(rows_bad)}', flush=True)
            except Exception as e:
                print(params.n, 'kernel', kern, 'dbg', dbg, 'ERR', e, flush=True)
    s.ctx.set_debug(0)
