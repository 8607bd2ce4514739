"""``python -m paper_2601_16637_b200 {solve,verify,bench} ...`` -- the reference CLI on the B200 backend."""

import sys

from .cli import main

sys.exit(main())
