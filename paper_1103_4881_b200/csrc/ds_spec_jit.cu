// ds_spec_jit.cu -- run-time compilation of K-N1s (ds_spec.cuh) for specs
// without a built-in instance.  (Stub: no JIT in this build.)
#include "ds.h"
#include "ds_internal.h"

namespace dsi {

SpecFn spec_jit_kernel(ds_handle*, int) { return nullptr; }

}  // namespace dsi
