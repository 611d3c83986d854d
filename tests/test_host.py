"""Host-side logic that needs no GPU: layout helpers, world validation,
process groups and ChunkedSequence validation (reference test_lasp2.py:226-240)."""
import numpy as np
import pytest
import torch

from paper_2502_07563_b200 import comm, shards
from paper_2502_07563_b200.lasp2 import ChunkedSequence


def test_split_pack_unpack_roundtrip():
    x = torch.arange(2 * 3 * 8 * 4, dtype=torch.float64).reshape(2, 3, 8, 4)
    parts = shards.split_chunks(x, 4)
    assert len(parts) == 4 and parts[1].shape == (2, 3, 2, 4)
    assert torch.equal(torch.cat(parts, dim=2), x)
    packed = shards.pack_slots(parts[2])
    assert packed.shape == (2 * 3 * 2, 4)
    assert torch.equal(shards.unpack_slots(packed, 2, 3), parts[2])
    with pytest.raises(ValueError):
        shards.split_chunks(x, 3)
    with pytest.raises(ValueError):
        shards.unpack_slots(packed, 5, 1)


def test_world_config_validation():
    assert comm.WorldConfig(4).sp_size == 4
    assert comm.WorldConfig(8, sp_size=4).dp_size == 2
    assert comm.WorldConfig(2, element_bytes=2).element_bytes == 2
    for bad in (dict(world_size=0), dict(world_size=4, sp_size=3), dict(world_size=2, element_bytes=3)):
        with pytest.raises(ValueError):
            comm.WorldConfig(**bad)


def test_process_groups_contiguous_sp_strided_dp():
    g = comm.process_groups(comm.WorldConfig(8, sp_size=4))
    assert g[5].sp_peers == (4, 5, 6, 7) and g[5].sp_position == 1
    assert g[5].dp_peers == (1, 5)


def test_chunked_sequence_validation_before_device():
    z = np.zeros((1, 1, 8, 4))
    with pytest.raises(ValueError):
        ChunkedSequence(z, z, z, 3)
    with pytest.raises(ValueError):
        ChunkedSequence(z, z, z[:, :, :4], 2)
    with pytest.raises(ValueError):
        ChunkedSequence(z[0], z[0], z[0], 1)
    with pytest.raises(ValueError):
        ChunkedSequence(z, z.astype(np.float32), z, 2)


def test_world_spawn_requires_cuda_when_absent():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        comm.world_spawn(comm.WorldConfig(2), lambda ctx: None)


def test_package_datagen_matches_pinned_oracle_generator():
    """The package's host generator (used for f64 reference data and weights) equals
    the oracle's, which test_oracle.py pins to the reference's golden values."""
    import numpy as np

    from oracle import lasp_oracle as O
    from paper_2502_07563_b200 import datagen

    for seed, tag in ((0, "q"), (1, "x/b0/h1"), (-3, ""), (2**70 + 5, "do")):
        for dt in (np.float64, np.float32):
            assert np.array_equal(datagen.gen_data(seed, 7, 5, tag, dt), O.gen_data(seed, 7, 5, tag, dt))
    assert np.array_equal(datagen.gen_slots(0, 2, 3, 9, 4, "k"), O.gen_slots(0, 2, 3, 9, 4, "k"))
    assert all(np.array_equal(a, b) for a, b in zip(datagen.qkv_slots(4, 1, 2, 8, 4), O.qkv_slots(4, 1, 2, 8, 4)))
    assert np.array_equal(datagen.projection_weight(7, 0, "q", 4), O.projection_weight(7, 0, "q", 4))
    assert datagen.projection_weight(7, 0, "q", 4)[0, 0] == 0.3980089845330995  # test_datagen.py:82
