"""python -m paper_2312_17396_b200 {eval,plan,compare,table1,verify} (__main__.py:1-5)."""
import sys

from .cli import main

sys.exit(main())
