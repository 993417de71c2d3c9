"""GPU: packed <-> padded bookkeeping (batching.hpp:20-27, 48-75) against numpy restatements and the reference's own
templates (through oracle/ref_shim.cpp)."""
import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S

pytestmark = pytest.mark.gpu


def np_packed_to_padded(packed, first, num, M, pad):
    out = np.full((len(num), M) + packed.shape[1:], pad, dtype=packed.dtype)
    for b, (f, n) in enumerate(zip(first, num)):
        out[b, :n] = packed[f:f + n]
    return out


def test_packed_padded_round_trip(cuda):
    from paper_2007_08501_b200.batching import item_to_element, packed_to_padded, padded_to_packed

    m = S.config_meshes("C2")
    fv = S.face_verts(m, S.bench_camera())
    first, num = m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    for arr, pad in ((fv, -7.5), (m.faces_packed(), -1), (m.faces_packed()[:, 0].astype(np.int32), 3),
                     (np.arange(len(fv) * 3, dtype=np.uint8).reshape(-1, 3), 9)):
        t = torch.as_tensor(np.ascontiguousarray(arr), device=cuda)
        got = packed_to_padded(t, first, num, pad_value=pad).cpu().numpy()
        want = np_packed_to_padded(arr, first, num, int(num.max()), pad)
        assert np.array_equal(got, want)
        back = padded_to_packed(torch.as_tensor(got, device=cuda), first, num, total=len(arr)).cpu().numpy()
        assert np.array_equal(back, arr)
    ite = item_to_element(first, num, len(fv) + 5, cuda).cpu().numpy()
    assert np.array_equal(ite[:len(fv)], np.repeat(np.arange(len(num)), num)) and np.all(ite[len(fv):] == -1)


def test_packed_padded_vs_reference_templates(reflib, cuda):
    """dr_packed_to_padded / dr_padded_to_packed / dr_packed_item_to_element vs the reference's own templates
    (batching.hpp:48-75, instantiated by oracle/ref_shim.cpp) on face_verts rows (9 doubles) and a scalar per
    face, including a zero-face mesh."""
    from paper_2007_08501_b200.batching import item_to_element, packed_to_padded, padded_to_packed

    m = S.config_meshes("C2")
    m.verts.insert(3, np.zeros((3, 3)))
    m.faces.insert(3, np.zeros((0, 3), dtype=np.int64))
    fv = S.face_verts(m, S.bench_camera())
    first, num = m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    offsets = np.concatenate([first, [first[-1] + num[-1]]])
    for arr, pad in ((fv.reshape(-1, 9), -7.5), (fv[:, 0, 2].copy(), 0.25)):
        want = reflib.packed_to_padded(arr, offsets, pad)
        got = packed_to_padded(torch.as_tensor(arr, device=cuda), first, num, pad_value=pad).cpu().numpy()
        assert np.array_equal(got.reshape(want.shape), want)
        back_ref, ite_ref = reflib.padded_to_packed(want, num)
        back = padded_to_packed(torch.as_tensor(got, device=cuda), first, num, total=len(arr)).cpu().numpy()
        assert np.array_equal(back.reshape(back_ref.shape), back_ref)
        assert np.array_equal(item_to_element(first, num, len(arr), cuda).cpu().numpy(), ite_ref)
