"""Long-horizon ring bookkeeping (BASELINE config 4: 10k frames = 834 blocks
of 12 frames): the device ring's integer replay (kvcache.RingIndex, used by
every engine Stage) must give, for every block, exactly the visible block
list of the reference rolling cache (kvcache.py:41-56; restated and pinned
in oracle.visible_schedule / attention_bruteforce's window rule), never
write the current block into a visible slot, and place the sink at i + delta
(kvcache.py:86-90) -- bit-exact integer checks, CPU only."""

import pytest

from oracle import livepipe_oracle as O
from paper_2512_04677_b200 import kvcache as K
from paper_2512_04677_b200.engine import EngineConfig

BLOCKS_10K_FRAMES = -(-10_000 // 12)  # 834 blocks


@pytest.mark.parametrize("capacity", [1, 2, 4, 8, 64])
def test_ring_replay_matches_reference_window(capacity):
    ring = K.RingIndex(capacity)
    sched = O.visible_schedule(BLOCKS_10K_FRAMES, capacity)
    for i in range(BLOCKS_10K_FRAMES):
        vis = [b for b, _ in ring.view()]
        assert vis == sched[i]
        mask = O.visible_mask(i, capacity)
        assert vis == [m for m in range(i) if mask[m]]
        slot = ring.write_slot(i)
        assert slot == i % (capacity + 1)
        assert slot not in {s for _, s in ring.view()}
        assert len(ring) <= capacity
        ring.push(i)


def test_ring_rejects_out_of_order():
    ring = K.RingIndex(2)
    ring.push(0)
    ring.push(1)
    with pytest.raises(ValueError, match="increasing"):
        ring.push(1)


@pytest.mark.parametrize("delta", [1, 3])
def test_sink_position_long_horizon(delta):
    assert [K.rolling_rope_index(i, delta) for i in (0, 1, 833)] == [delta, 1 + delta, 833 + delta]
    with pytest.raises(ValueError):
        K.rolling_rope_index(5, 0)


def test_keys_per_block_steady_state():
    # N_kv = S + L*N + N once the ring is full (24,960 at 480p, L=4)
    from paper_2512_04677_b200.model import WAN_14B

    n = 3 * WAN_14B.tokens_per_frame
    ring = K.RingIndex(4)
    for i in range(10):
        ring.push(i)
    assert WAN_14B.tokens_per_frame + len(ring) * n + n == 24_960
    assert EngineConfig(mode="tpp", blocks=BLOCKS_10K_FRAMES).total_frames == BLOCKS_10K_FRAMES * 12
