// ssb_summary.cu — placeholder (implemented next)
#include "../../include/ssb.h"
extern "C" size_t ssb_summary_work_bytes(const ssb_summary_group*, int32_t) { return 0; }
extern "C" int32_t ssb_summarize(ssb_trace, ssb_records, const ssb_summary_group*, const ssb_summary_group*, int32_t,
                                 ssb_summary*, void*, size_t, void*) { return SSB_E_ARG; }
