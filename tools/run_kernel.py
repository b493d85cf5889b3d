"""Run one full-size bench kernel a few times in-process (for ncu captures).

usage: python tools/run_kernel.py gamma|dirichlet|gibbs|gibbs1|gaussian|uniform [reps]
(the same workloads as tools/variant_time.py, without the subprocess layer)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import variant_time  # noqa: E402

code = variant_time.CHILD.replace("ROOT", repr(ROOT)).replace("WHAT", repr(sys.argv[1]))
exec(compile(code, "variant_child", "exec"))
