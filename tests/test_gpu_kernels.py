"""GPU parity of the standalone kernels through the C ABI: K1 gradgen (bit-exact vs the
reference GradGen golden vectors and the oracle) and K4 reduce+SGD (bit-exact vs the
reference ShardState fixtures and the oracle)."""

import hashlib

import numpy as np
import pytest

import p3_oracle as O

pytestmark = pytest.mark.gpu


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def test_gradgen_golden_values(cuda, golden):
    from paper_1905_03960_b200.hashing import gradient_value

    for args, bits in golden["gradient_values"]:
        assert int(np.float32(gradient_value(*args)).view(np.uint32)) == bits, args


def test_gradgen_golden_blocks(cuda, golden):
    from paper_1905_03960_b200.hashing import gradient_block

    for args, h in golden["gradient_blocks"]:
        got = gradient_block(*args)
        assert got.dtype == np.float32 and len(got) == args[4]
        assert sha(got.astype("<f4").tobytes()) == h, args


@pytest.mark.parametrize("start,count", [(0, 1), (3, 5), (1, 4099), (7, 50_000), (0, 2_000_001)])
@pytest.mark.parametrize("misalign", [0, 1, 3])
def test_gradgen_vs_oracle_misaligned(cuda, start, count, misalign):
    import torch

    from paper_1905_03960_b200.hashing import gradient_block_device

    buf = torch.full((count + 8,), 7.0, device="cuda")
    gradient_block_device(2**63 + 5, 11, 9, start, count, out=buf[misalign : misalign + count])
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    assert host[misalign : misalign + count].tobytes() == O.grad_block(2**63 + 5, 11, 9, start, count).tobytes()
    assert (host[:misalign] == 7.0).all() and (host[misalign + count :] == 7.0).all()


def test_gradgen_large_layer(cuda):
    # VGG-19 fc6 size: full-layer generation on the device, spot-checked against the oracle
    from paper_1905_03960_b200.hashing import gradient_block_device

    n = 102_760_448
    g = gradient_block_device(19, 3, 32, 0, n).cpu().numpy()
    for lo in (0, 12_345_677, n - 4099):
        assert g[lo : lo + 4099].tobytes() == O.grad_block(19, 3, 32, lo, 4099).tobytes()
    assert -0.001 < float(g.mean()) < 0.001


def _update_case(case):
    rng = np.random.RandomState(1000 + case)
    n = int(rng.randint(1, 70_000)) if case % 4 == 0 else int(rng.randint(1, 300))
    nw = int(rng.randint(1, 9))
    lr = float(rng.uniform(0.0, 1.0))
    params = rng.uniform(-5, 5, n).astype(np.float32)
    grads = {r: rng.uniform(-3, 3, n).astype(np.float32) for r in range(nw)}
    return n, nw, lr, params, grads


def test_shard_update_reference_fixtures(cuda, golden):
    from paper_1905_03960_b200.plan import SliceKey
    from paper_1905_03960_b200.server import ShardState

    for case, n, nw, lr, h in golden["shard_updates"]:
        _, _, _, params, grads = _update_case(case)
        s = ShardState(SliceKey(1, 2), params.copy(), nw, lr)
        for r in range(nw):
            assert s.on_push(r, 0, grads[r]) == (r == nw - 1)
        got = s.aggregate_and_update()
        assert sha(got.astype("<f4").tobytes()) == h, case
        assert s.iteration == 1 and not s.pending


@pytest.mark.parametrize("nw", [1, 2, 3, 5, 7, 8, 11, 16])
@pytest.mark.parametrize("offset", [0, 1])
def test_shard_update_vs_oracle(cuda, nw, offset):
    import torch

    from paper_1905_03960_b200.server import shard_update_device

    rng = np.random.RandomState(nw * 10 + offset)
    n = 200_003
    params = rng.uniform(-5, 5, n).astype(np.float32)
    grads = {r: (rng.uniform(-3, 3, n) * 10.0 ** rng.randint(-8, 8, n)).astype(np.float32) for r in range(nw)}
    pbuf = torch.zeros(n + 1, device="cuda")
    pbuf[offset : offset + n] = torch.from_numpy(params).cuda()
    gd = [torch.from_numpy(grads[r]).cuda() for r in range(nw)]
    shard_update_device(pbuf[offset : offset + n], gd, 0.37)
    torch.cuda.synchronize()
    want = O.shard_update(params, grads, 0.37)
    assert pbuf[offset : offset + n].cpu().numpy().tobytes() == want.tobytes()


def test_shard_update_signed_zero_and_lr0(cuda):
    from paper_1905_03960_b200.plan import SliceKey
    from paper_1905_03960_b200.server import ShardState

    # -0.0 gradients: the reference starts from +0.0 so the sum is +0.0
    s = ShardState(SliceKey(0, 0), np.array([0.0, -0.0, 1.0], np.float32), 2, 0.5)
    s.on_push(0, 0, np.array([-0.0, -0.0, 2.0], np.float32))
    s.on_push(1, 0, np.array([-0.0, 0.0, 2.0], np.float32))
    want = O.shard_update(np.array([0.0, -0.0, 1.0], np.float32),
                          {0: np.array([-0.0, -0.0, 2.0], np.float32), 1: np.array([-0.0, 0.0, 2.0], np.float32)}, 0.5)
    assert s.aggregate_and_update().tobytes() == want.tobytes()
    # lr = 0 conserves parameters (tests/test_server.py:103-111)
    rng = np.random.RandomState(3)
    params = rng.uniform(-2, 2, 16).astype(np.float32)
    s = ShardState(SliceKey(0, 0), params.copy(), 2, 0.0)
    for k in range(3):
        s.on_push(0, k, rng.uniform(-1, 1, 16).astype(np.float32))
        s.on_push(1, k, rng.uniform(-1, 1, 16).astype(np.float32))
        assert s.aggregate_and_update().tobytes() == params.tobytes()


def test_shard_protocol_errors(cuda):
    from paper_1905_03960_b200.plan import SliceKey
    from paper_1905_03960_b200.proto import ProtocolError
    from paper_1905_03960_b200.server import ShardState

    s = ShardState(SliceKey(0, 0), np.zeros(4, np.float32), 2, 0.1)
    with pytest.raises(ProtocolError, match="iteration"):
        s.on_push(0, 3, np.zeros(4, np.float32))
    with pytest.raises(ProtocolError, match="rank"):
        s.on_push(5, 0, np.zeros(4, np.float32))
    with pytest.raises(ProtocolError, match="length"):
        s.on_push(0, 0, np.zeros(3, np.float32))
    s.on_push(0, 0, np.zeros(4, np.float32))
    with pytest.raises(ProtocolError, match="duplicate"):
        s.on_push(0, 0, np.zeros(4, np.float32))
    with pytest.raises(ProtocolError, match="aggregate"):
        s.aggregate_and_update()


@pytest.mark.parametrize("nw", [1, 3, 4])
def test_shard_update_momentum(cuda, nw):
    # extension (not in the reference): v = mu*v + mean(g); p -= lr*v, every op rounded
    import torch

    from paper_1905_03960_b200.server import shard_update_device

    rng = np.random.RandomState(nw)
    n = 10_007
    p = rng.uniform(-1, 1, n).astype(np.float32)
    v = rng.uniform(-1, 1, n).astype(np.float32)
    grads = {r: rng.uniform(-1, 1, n).astype(np.float32) for r in range(nw)}
    pd, vd = torch.from_numpy(p).cuda(), torch.from_numpy(v).cuda()
    shard_update_device(pd, [torch.from_numpy(grads[r]).cuda() for r in range(nw)], 0.3, momentum=0.9, momentum_buf=vd)
    acc = np.zeros(n, np.float32)
    for r in range(nw):
        acc = acc + grads[r]
    g = acc / np.float32(nw)
    v2 = np.float32(0.9) * v + g
    p2 = p - np.float32(0.3) * v2
    assert vd.cpu().numpy().tobytes() == v2.astype(np.float32).tobytes()
    assert pd.cpu().numpy().tobytes() == p2.astype(np.float32).tobytes()
