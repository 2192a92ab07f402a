// logan_fmt_2bit_z.cu — run_batch<LOGAN_SEQ_2BIT | FMT_Z> and every kernel it launches (one format
// per translation unit: the build compiles them in parallel). See logan_impl.cuh.
#include "logan_impl.cuh"

namespace logan {
template LOGAN_RUN_BATCH_SIG(LOGAN_SEQ_2BIT | FMT_Z);
}  // namespace logan
