// logan_fmt_u8s_z.cu — run_batch<FMT_U8S | FMT_Z> and every kernel it launches (one format
// per translation unit: the build compiles them in parallel). See logan_impl.cuh.
#include "logan_impl.cuh"

namespace logan {
template LOGAN_RUN_BATCH_SIG(FMT_U8S | FMT_Z);
}  // namespace logan
