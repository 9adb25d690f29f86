import sys, time, faulthandler
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, oracle
from golden_util import load, case_trace, policy_name, GOLDEN
import paper_2601_17063_b200 as mcb
from paper_2601_17063_b200 import engine, _lib
from test_parity_gpu import to_trace, code_of, cost_of
mode = sys.argv[1]
_lib.set_tuning(_lib.MCB_TUNE_SOLO_MIN, 0 if mode == "solo" else 1 << 62)
for ci, case in enumerate(load("small_cases.json.gz")["cases"][:8]):
    header, events = case_trace(case)
    L, E, K = header
    packed = mcb.pack_trace(to_trace(header, events))
    for run in case["runs"]:
        if policy_name(run["policy"]) != "ml": continue
        nets = oracle.nets_from_spec(run["nets"], L, E, GOLDEN)
        print(ci, case["name"], packed.uniform, run["policy"], run["capacity"], flush=True)
        res = engine.replay_host(packed, [code_of(run["policy"])], [run["capacity"]], cost_of(run["cost"]), run["window"], nets)
        print("  ok", res["reports"][0,0,0].tolist(), flush=True)
