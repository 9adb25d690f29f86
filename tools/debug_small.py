import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
from golden_util import load, case_trace, policy_name
import paper_2601_17063_b200 as mcb
from paper_2601_17063_b200 import engine, _lib
from test_parity_gpu import to_trace, code_of, cost_of
case = load("small_cases.json.gz")["cases"][int(sys.argv[1]) if len(sys.argv) > 1 else 0]
header, events = case_trace(case)
packed = mcb.pack_trace(to_trace(header, events))
print(case["name"], header, packed.uniform, packed.total_acc, packed.acc[:packed.total_acc])
for run in case["runs"][:3]:
    res = engine.replay_host(packed, [code_of(run["policy"])], [run["capacity"]], cost_of(run["cost"]), run["window"], None, want_outcomes=True)
    print(run["policy"], run["capacity"], res["reports"][0,0,0], res["outcomes"][0,0,:packed.total_acc])
    print("want", run["decisions"])
