"""`python -m paper_2512_07350_b200 SUBCOMMAND --config PATH ...` — the reference's `lpsim`
CLI (tools/lpsim_main.cpp) on the B200 engine; same as the native paper_2512_07350_b200/lpsim_b200."""
import sys

from . import lp

sys.exit(lp.cli(sys.argv[1:]))
