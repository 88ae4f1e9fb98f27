import os, sys, runpy
sys.path.insert(0, "/root/repo")
m = runpy.run_path("/root/repo/scripts/learn_trace.py", run_name="lt")
m["run"]("dbg=" + os.environ.get("SP_LEARN_DBG", "0"), 200, num_columns=1024, synapses_per_column=256)
