"""Run bench.py with a stall watchdog: after LP_WATCH_S seconds, dump every thread's Python stack
to stderr and exit (diagnoses intermittent hangs).  usage: python scripts/bench_watch.py [bench args]"""
import faulthandler
import os
import runpy
import sys

faulthandler.dump_traceback_later(int(os.environ.get("LP_WATCH_S", "120")), exit=True)
sys.argv = ["bench.py"] + sys.argv[1:]
sys.path.insert(0, os.getcwd())
runpy.run_path("bench.py", run_name="__main__")
