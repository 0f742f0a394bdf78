// generated: explicit instantiation of the L = 2^14 engine
#include "../tsf_dispatch_impl.cuh"

template struct tsf::Dispatch<14>;
