"""CPU-side checks of the torch-mode wrapper's construction logic (no GPU needed)."""

import inspect

from paper_1905_03960_b200 import ddp


def test_p3_dataparallel_signature_complete():
    # every keyword the constructor forwards must be a parameter (catches NameErrors early)
    src = inspect.getsource(ddp.P3DataParallel.__init__)
    params = set(inspect.signature(ddp.P3DataParallel.__init__).parameters)
    for name in ("push_dtype", "drain_bytes", "pub_batch_bytes", "drain_linger_us", "finish_ctas", "throttle_bps",
                 "plan_mode", "priority_mode", "momentum", "max_slice", "comm_ctas"):
        assert name in params, name
        assert name in src


def test_dense_layout_helper():
    import torch

    assert ddp._dense(torch.empty(4, 3, 2, 2))
    assert ddp._dense(torch.empty(4, 3, 2, 2).to(memory_format=torch.channels_last))
    assert not ddp._dense(torch.empty(4, 6)[:, ::2])
