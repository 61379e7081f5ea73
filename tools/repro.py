import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2604_08706_b200 as rb
from tests.test_gpu_parity import make_record
b = rb.ShardedReplayBuffer(1, 3)
print("created", flush=True)
print(b.push(make_record(1)), flush=True)
