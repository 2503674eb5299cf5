// engine_cols.cu -- the analysis kernel compiled a second time, for inputs whose resource
// ids come as a res column, with the tile geometry measured best for them: 11 compute
// warps x 15 records.  A/B on one B200, kernel ms, res-column layout (tools/ab.py): C5
// 7.30 -> 6.99, C3 2.09 -> 1.85, C2 0.371 -> 0.375; the CSR layout keeps 15 x 11 (C5 7.38
// vs 7.63).  Also measured with 3-stage rings (11 x 9, 7 x 15, 9 x 11): C5 8.1-8.6 ms.
// capi.cu picks the compilation per call and sizes the call's tiles, look-back slots and
// error-path scratch with that compilation's tile (tile_records()).
// (HB_COLS_* override the geometry for tuning builds, tools/build_engine_variants.sh.)
#ifndef HB_COLS_WARPS
#define HB_COLS_WARPS 11
#endif
#ifndef HB_COLS_ITEMS
#define HB_COLS_ITEMS 15
#endif
#ifndef HB_COLS_STAGES
#define HB_COLS_STAGES 2
#endif
#define HB_WARPS HB_COLS_WARPS
#define HB_ITEMS HB_COLS_ITEMS
#define HB_STAGES HB_COLS_STAGES
#define HB_ENGINE_NS hb_cols
#include "engine.cu"
