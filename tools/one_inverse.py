import sys
sys.path.insert(0, ".")
import torch
from paper_1307_2665_b200 import _native
lib = _native.load()
n = int(sys.argv[1]); batch = int(sys.argv[2])
A = torch.randn(batch, n, n, dtype=torch.float64, device="cuda") + n * torch.eye(n, dtype=torch.float64, device="cuda")
ws = torch.empty(lib.hps_inverse_workspace_bytes(n, batch), dtype=torch.uint8, device="cuda")
st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
for _ in range(2):
    X = A.clone()
    _native.check(lib.hps_inverse_batched(_native.context(), n, batch, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(), _native.ptr(st), _native.stream_ptr()), "inv")
torch.cuda.synchronize(); print("ok")
