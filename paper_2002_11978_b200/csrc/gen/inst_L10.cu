// generated: explicit instantiation of the N_mv = 2^10 engine
#include "../tsf_dispatch_impl.cuh"

template struct tsf::Dispatch<10>;
