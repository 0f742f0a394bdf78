// LargeDispatch instantiation, one size per translation unit (parallel build).
#include "../tsf_large_impl.cuh"

template struct tsf::LargeDispatch<7>;
