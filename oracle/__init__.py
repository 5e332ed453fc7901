"""FlashNorm oracle package — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything under oracle/.  The product package
paper_2407_09577_b200 never imports it; the two share no code.

* flashnorm_oracle.py : plain fp64 definitions from PAPER.md (the parity target)
* fold_mirror.py      : CPU folds in the same precision/order as the CUDA folds
                        (the bit-exact target for the fold kernels)
"""
from . import flashnorm_oracle, fold_mirror  # noqa: F401
