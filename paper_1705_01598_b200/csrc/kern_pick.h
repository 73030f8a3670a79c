// kern_pick.h -- kernel instantiation lookup, one function per translation
// unit (kernels_tile.cu, kernels_sd.cu, kernels_2d.cu, kernels_vg.cu), used
// by the launch layer (kernels.cu).  nullptr = no such instantiation.
#pragma once

namespace tt {

const void* pick_copy();
const void* pick_tile(int esize, int nreg, bool idx64);
const void* pick_tile_acc(int esize, int nreg);
const void* pick_tile_async(int esize, int nreg, bool idx64);
const void* pick_tile_sd(int esize, int q, int r, int stages);
const void* pick_rowcopy(int esize, bool idx64);
const void* pick_tiled2d(int esize, int vec, int ta, int tb, bool idx64);
const void* pick_tiled2d_async(int esize, int ta, int tb, int stages);
const void* pick_tile_vg(int esize, int nreg, int items, int stages, int threads);
const void* pick_tiled2d_tma(int esize, int rank);

}  // namespace tt
