// Shape of the patch-12 stride-4 strip kernel (reference rows per strip, dy per block, warps
// per strip).  c2 (512^2, 15,876 references) fills only part of the GPU, so shorter strips
// (more warps) win: 2/8/2 369 us, 2/12/2 386, 2/4/2 459, 1/8/1 463, 2/6/2 427, 4/4/2 535,
// 4/8/2 530, 1/4/1 582.
#pragma once
#ifndef GBM3D_S12_TRY
#define GBM3D_S12_TRY 2
#endif
#ifndef GBM3D_S12_D
#define GBM3D_S12_D 8
#endif
#ifndef GBM3D_S12_WPS
#define GBM3D_S12_WPS 2
#endif
