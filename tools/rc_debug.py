import sys, os
sys.path.insert(0, ".")
from types import SimpleNamespace as NS
import numpy as np
import paper_2406_01939_b200 as P
from oracle.oracle import ORC
J, I, T, M = 10, 300, 20000, 512
ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, 7))
inst = P.Instance(ons.nodes, ons.products, ons.horizon, ons.product, ons.reward_row, ons.reward_table, ons.capacity, ons.inventory)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_partition(inst, M, 1)
r = P.picard_simulate(inst, pol, plan, P.PicardConfig(record_trace=True))
print(r.conflicts, r.timing)
