"""Host logic of the peer-memory factor aggregation (comm.peer_layout, csrc/peer.cu): the byte layout every
rank gives its CUDA-IPC allocation, and the alignment the 16-byte push path relies on.  No GPU needed."""
from paper_2107_06533_b200 import schedule as S
from paper_2107_06533_b200.comm import peer_layout


def test_layout_regions_disjoint_and_aligned():
    for world in (2, 3, 4, 8):
        for sizes in ({"A": 1, "G": 1}, {"A": 12345, "G": 777}, {"A": 45_000_001, "G": 3_000_003}):
            off, stride, total = peer_layout(world, sizes, n_slots=37, extra=999)
            assert off["A"] >= 37 * world * 4  # flags first
            assert off["A"] + world * stride["A"] * 4 <= off["G"]
            assert off["G"] + world * stride["G"] * 4 <= off["X"]
            assert off["X"] + 999 * 4 <= total
            for k in ("A", "G", "X"):
                assert off[k] % 256 == 0
            for k in ("A", "G"):
                assert stride[k] >= sizes[k] and stride[k] % 64 == 0


def test_inbox_rows_co_aligned_with_fusion_buffer():
    # element s of row q sits at the same address mod 16 as element s of a 256-aligned fusion buffer
    a_dims = [147, 576, 1152, 2304, 4608, 64, 2048]
    g_dims = [64, 64, 128, 256, 512, 2048, 1000]
    a_off, g_off, size_a, size_g = S.packed_layout(a_dims, g_dims)
    off, stride, _ = peer_layout(4, {"A": size_a, "G": size_g}, n_slots=9)
    for kind, offs in (("A", a_off), ("G", g_off)):
        for q in range(4):
            for s in offs:
                addr = off[kind] + (q * stride[kind] + s) * 4
                assert addr % 16 == (s * 4) % 16
