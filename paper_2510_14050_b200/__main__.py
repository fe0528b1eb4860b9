"""python -m paper_2510_14050_b200 {generate,analyze,bench} (the reference's `netmeter` CLI)."""
import sys

from .cli import main

sys.exit(main())
