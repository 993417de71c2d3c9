"""Work counters of the fine stage (debug build with -DDR_STATS=1, loaded through DR_RASTER_LIB).

  DR_RASTER_LIB=build/variants/stats/libdr_raster_b200.so python tools/fine_stats.py C4 [C5 ...]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2007_08501_b200 import _lib, rasterize_meshes, scenes as S  # noqa: E402
sys.path.insert(0, ROOT)
from bench import config_settings  # noqa: E402

NAMES = ["list entries scanned", "faces staged", "pairs enumerated", "pairs evaluated (not z-culled)",
         "pairs passing", "micro-tiles", "(unused)", "pair steps", "candidates merged (register path)",
         "merge calls (warps)", "merged below the list tail", "overflow merges (warps)"]


def main():
    L = _lib.load()
    fn = L.dr_debug_stats
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    dev = torch.device("cuda:0")
    for cfg in sys.argv[1:] or ["C4"]:
        m = S.config_meshes(cfg)
        cam = S.bench_camera()
        fv = torch.as_tensor(S.face_verts(m, cam), device=dev)
        first = torch.as_tensor(m.mesh_to_face_first_idx(), device=dev)
        num = torch.as_tensor(m.num_faces_per_mesh(), device=dev)
        rs = config_settings(cfg)
        out = (C.c_ulonglong * 12)()
        fn(out, 1)
        p2f = rasterize_meshes(fv, first, num, rs)[0]
        torch.cuda.synchronize()
        fn(out, 1)
        occ = int((p2f >= 0).sum())
        print(f"{cfg}: occupied slots {occ:,}")
        for n, v in zip(NAMES, out):
            print(f"  {n:32s} {v:16,d}")


if __name__ == "__main__":
    main()
