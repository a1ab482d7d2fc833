"""CPU oracle for the compensated Yee operator and its smallest eigenvalues.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2511_17107_b200``) never imports it and shares no code with it.

See ``oracle/pc_oracle.py`` for the functions; each cites the PAPER.md passage it follows.
"""
from .pc_oracle import *  # noqa: F401,F403
