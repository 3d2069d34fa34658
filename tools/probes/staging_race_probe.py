import contextlib, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_2007_14152_b200 import engine
orig = engine._stage_buffers
def nolock(torch, dev):
    b, v, p, _ = orig(torch, dev)
    return b, v, p, contextlib.nullcontext()
engine._stage_buffers = nolock
import test_gpu_parity as t
try:
    t.test_concurrent_staged_transfers_and_infer(True)
    print("without the lock: test passed (race not caught)")
except AssertionError as e:
    print("without the lock: test FAILED as expected", repr(e)[:200])
