import json, sys, os, traceback
sys.path.insert(0, os.getcwd())
from paper_2405_16256_b200 import planner
cases = json.load(open('tests/golden/search_cases.json'))
for c in cases:
    if c["name"] in ("C3pp12-full",):
        for log in (False, True):
            try:
                o = planner.search(c["docs"], log=log)
                print(c["name"], log, o.iteration_time_s, o.candidates_simulated, o.candidates_pruned, len(o.log), c["candidates_simulated"], c["candidates_pruned"])
            except Exception as e:
                print(c["name"], log, "ERR", e)
