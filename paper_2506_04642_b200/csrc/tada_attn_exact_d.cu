// K2-exact v2 instantiations for head_dim 32 / 64 / 256 (the kernel: tada_attn_exact2.cuh).
#include "tada_attn_exact2.cuh"

namespace tada {

template <int BITS>
static int launch_d(const AttnArgs& a, int batch, const exact2::Plan& pl, cudaStream_t st) {
  switch (a.L.head_dim) {
    case 32: return exact2::launch_g<BITS, 32>(a, batch, pl, st);
    case 64: return exact2::launch_g<BITS, 64>(a, batch, pl, st);
    default: return exact2::launch_g<BITS, 256>(a, batch, pl, st);
  }
}

int exact2_launch_other_d(const AttnArgs& a, int batch, const exact2::Plan& pl, cudaStream_t st) {
  switch (a.L.bits) {
    case 2: return launch_d<2>(a, batch, pl, st);
    case 4: return launch_d<4>(a, batch, pl, st);
    case 8: return launch_d<8>(a, batch, pl, st);
    default: return launch_d<16>(a, batch, pl, st);
  }
}

}  // namespace tada
