import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_controller as T
orig = torch.allclose
def ac(a, b, rtol=0, atol=0):
    print("rel diff", float((a - b).abs().max() / a.abs().max()), tuple(a.shape))
    return True
torch.allclose = ac
for i in range(2):
    T.test_saved_tensor_hooks_free_memory_and_retain_graph(None)
print("done")
