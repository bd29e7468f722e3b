"""TEST INFRASTRUCTURE ONLY -- the plain fp64 CPU oracle of the PFPG / PFAM hot path.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import this package.  The product (`paper_1904_10585_b200`) never imports it and
shares no code with it; the only common dependency is the seeded input module `pfinputs`.
"""
from .pf_oracle import *  # noqa: F401,F403
from .pf_svt import *  # noqa: F401,F403,E402
