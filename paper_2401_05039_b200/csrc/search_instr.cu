// search_instr.cu — the instrumented instantiation of the search kernel (MBE_STATS phase
// counters, per-root counters, bounded listing).  Same source as search.cu.
#define MBE_INSTR 1
#include "search.cu"
