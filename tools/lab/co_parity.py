"""K8c (co-resident decode attention) inside the tiny-model serving replay WITHOUT the row
split: every decode attention call of the run goes to K8c (hy_set_decode_coresident on the
driver thread).  Lab triage for the split-mode parity failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity_util import oracle_replay  # noqa: E402
import test_parity_gpu as T  # noqa: E402
from paper_2505_12658_b200 import _lib, get_shape  # noqa: E402

lib = _lib.load()
lib.hy_set_decode_coresident(int(os.environ.get("CO", "1")))
shape = get_shape("tiny")
g, cl, _ = T._run("config1_2000rps", shape)
res = oracle_replay(cl, shape, seed=0)
print({k: res[k] for k in ("max_abs_err", "rows", "tokens_equal", "near_ties")})
