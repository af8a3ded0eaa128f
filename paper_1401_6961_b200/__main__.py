"""`python -m paper_1401_6961_b200 [flags]`: the run-report / scaling-series harness
(harness.py; the reference CLI's flags, cli.py:266-351)."""
import sys

from .harness import main

sys.exit(main())
