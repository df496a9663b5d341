"""CPU oracle for RHOSVD C2T.  TEST INFRASTRUCTURE ONLY: importable from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
The product package paper_2201_12663_b200 never imports this package."""
from .rhosvd_oracle import *  # noqa: F401,F403
from .compare import *  # noqa: F401,F403
from .t2c_oracle import *  # noqa: F401,F403
from .rs_oracle import *  # noqa: F401,F403
from .als_oracle import *  # noqa: F401,F403
from .conv_oracle import *  # noqa: F401,F403
