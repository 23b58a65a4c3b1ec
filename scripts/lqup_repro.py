"""Reproduce an LQUP fuzz failure under feature knobs.  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
from test_gpu_lqup import _check_valid  # noqa: E402

torch.cuda.set_device(0)
for (p, m, n, seed) in [(2, 844, 341, 1), (3, 572, 532, 2), (29, 423, 836, 3), (2, 634, 563, 4), (2, 300, 300, 5),
                        (3, 700, 700, 6), (5, 1000, 1000, 7)]:
    rng = np.random.default_rng(seed)
    A = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    want_r, _ = oracle.rank_det(p, A)
    res = []
    for knobs in [{}, {"FF_LQUP_GROUP": "1"}, {"FF_SMALL": "0"}, {"FF_LQUP_NOSPEC": "1"},
                  {"FF_LQUP_GROUP": "1", "FF_SMALL": "0"}]:
        for kk, vv in knobs.items():
            os.environ[kk] = vv
        dA = torch.from_numpy(A).cuda()
        Q, P, rk = ff.lqup(p, dA)
        torch.cuda.synchronize()
        ok = rk == want_r
        if ok:
            try:
                _check_valid(p, A, dA.cpu().numpy(), Q, P, rk)
            except AssertionError:
                ok = False
        res.append("%s:%s" % (",".join("%s=%s" % kv for kv in knobs.items()) or "default", "ok" if ok else "BAD(r=%d want %d)" % (rk, want_r)))
        for kk in knobs:
            del os.environ[kk]
    print("p=%d m=%d n=%d: %s" % (p, m, n, "  ".join(res)), flush=True)
