"""Library cross-check (PAPER.md:104 chain reduction): a chain-shaped tree through stree_tree_scan
and stree_commit must equal the ordinary Mamba-2 recurrence as an independent library implements it — vLLM's
`selective_state_update` (the per-token SSM state update of its Mamba-2 decode path), applied token by token.

Test infrastructure only: the library is called here, never on the product path.  Skipped when vLLM (or its
Triton kernels) is not importable on the box."""
import numpy as np
import pytest
import torch

from gen import inputs, trees
from tests.helpers import TOL_BF16, assert_h_close, assert_y_close

pytestmark = pytest.mark.gpu


def _vllm_update():
    try:
        from vllm.model_executor.layers.mamba.ops.mamba_ssm import selective_state_update
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"vLLM selective_state_update not importable: {e}")
    return selective_state_update


@pytest.mark.parametrize("B,T,H,G", [(2, 16, 8, 2), (1, 40, 24, 1)])
def test_chain_scan_and_commit_match_vllm_selective_state_update(B, T, H, G):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ssu = _vllm_update()
    from paper_2505_14969_b200 import api
    P, N = 64, 128
    par = np.stack([trees.chain(T)] * B)
    prob = inputs.make_problem(inputs.Dims(B, T, H, P, N, G, "bf16"), par, seed=1234 + T)
    t = api.upload(prob)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = api.tree_scan(t, st)
    path = torch.from_numpy(np.tile(np.arange(T, dtype=np.int32), (B, 1))).cuda()
    plen = torch.full((B,), T, dtype=torch.int32, device="cuda")
    h_new = api.commit(t, path, plen, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0

    # the same values (bf16 inputs widened exactly) through the library, one token at a time, fp32 state
    dev = torch.device("cuda")
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
    x, Bm, Cm = f32(prob.io_as_f32("x")), f32(prob.io_as_f32("Bm")), f32(prob.io_as_f32("Cm"))
    dt, A, D = f32(prob.dt), f32(prob.A), f32(prob.D)
    state = f32(prob.h0).clone()                                  # [B][H][P][N]
    A_e = A[:, None, None].expand(H, P, N)
    D_e = D[:, None].expand(H, P)
    bias = torch.zeros(H, P, dtype=torch.float32, device=dev)
    ys = []
    for i in range(T):
        out = torch.empty(B, H, P, dtype=torch.float32, device=dev)
        ssu(state, x[:, i].contiguous(), dt[:, i, :, None].expand(B, H, P), A_e, Bm[:, i].contiguous(),
            Cm[:, i].contiguous(), D_e, bias, dt_softplus=False, out=out)
        ys.append(out)
    torch.cuda.synchronize()
    y_lib = torch.stack(ys, dim=1).cpu().numpy().astype(np.float64)   # [B][T][H][P]
    assert_y_close(y.float().cpu().numpy(), y_lib, TOL_BF16)
    assert_h_close(h_new.cpu().numpy(), state.cpu().numpy().astype(np.float64), 1e-4)
