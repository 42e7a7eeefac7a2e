"""Run config-4 evaluations with SSUM_TRACE=1 (host phase breakdown on stderr)."""
import os
import sys

os.environ["SSUM_TRACE"] = "1"
sys.argv = [sys.argv[0], "5"] + sys.argv[1:]
exec(open(os.path.join(os.path.dirname(__file__), "profile_step.py")).read())
