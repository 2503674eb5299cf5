// engine_long.cu -- the analysis kernel compiled a third time, for res-column inputs whose
// devices hold long record runs (>= kLongRun records per device on average): 8 compute
// warps x 19 records.  A/B on one B200, kernel ms, res-column layout (tools/ab.py; 11 x 15 in
// parentheses): C4 3.23 (3.66), C3 1.66 (1.76), but C5 7.08 (6.94) and C2 0.401 (0.376) --
// hence the choice by run length in capi.cu (C3 / C4: ~4.4e5 - 4.9e5 records per device;
// C2 / C5: 4.9e4 - 6.1e4).
#define HB_WARPS 8
#define HB_ITEMS 19
#define HB_ENGINE_NS hb_long
#include "engine.cu"
