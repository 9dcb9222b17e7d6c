"""`python -m paper_2411_09287_b200 <command> ...` -- the ring3pc CLI."""

import sys

from .cli import main

sys.exit(main())
