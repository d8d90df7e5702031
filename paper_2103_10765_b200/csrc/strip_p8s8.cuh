// Shape of the stride-8 strip kernel (reference rows per strip, dy per block, warps per strip):
// solo warps, one reference row, 8 dy per block (c3-size image, r19 K16: 1.07 ms; 2/4/2 1.44,
// 2/8/2 1.10, 1/4/1 1.37; the direct kernel 6.6 ms).
#pragma once
#ifndef GBM3D_S8_TRY
#define GBM3D_S8_TRY 1
#endif
#ifndef GBM3D_S8_D
#define GBM3D_S8_D 8
#endif
#ifndef GBM3D_S8_WPS
#define GBM3D_S8_WPS 1
#endif
