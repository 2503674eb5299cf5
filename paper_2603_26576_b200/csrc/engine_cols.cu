// engine_cols.cu -- the analysis kernel compiled a second time, for inputs whose resource
// ids come as a res column, with the tile geometry measured best for them: 11 compute
// warps x 15 records (the same 5280-record tile as the default 15 x 11, so tile counts and
// the workspace layout are shared).  A/B on one B200, kernel ms, res-column layout
// (tools/ab.py): C5 7.30 -> 6.99, C3 2.09 -> 1.85, C2 0.371 -> 0.375; the CSR layout keeps
// 15 x 11 (C5 7.38 vs 7.63).  capi.cu picks the compilation per call.
#define HB_WARPS 11
#define HB_ITEMS 15
#define HB_ENGINE_NS hb_cols
#include "engine.cu"
