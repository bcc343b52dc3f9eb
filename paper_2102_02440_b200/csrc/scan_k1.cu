// scan_k1.cu — k_scan instances with 1 key column(s) (see scan_kernel.cuh).
#include "scan_kernel.cuh"

namespace {

typedef void (*ScanKernel)(const SParams);

template <int NK, int NP>
static ScanKernel pick_kw(int kw, bool fast, int sub, bool t3) {
    if (t3) return k_scan<NK, NP, 0, false, 1, true>;   // 3-D tensor targets: generic hashing drain
    if constexpr (NK <= 2 && NP <= 2) {
        if (fast) {
            if (NP == 0) return k_scan<NK, NP, 0, true, 1, false>;
            if (kw == 4) return sub == 4 ? k_scan<NK, NP, 4, true, 4, false> : k_scan<NK, NP, 4, true, 1, false>;
        }
    }
    if (NP == 0) return k_scan<NK, NP, 0, false, 1, false>;
    return kw == 4 ? k_scan<NK, NP, 4, false, 1, false> : kw == 8 ? k_scan<NK, NP, 8, false, 1, false> : k_scan<NK, NP, 0, false, 1, false>;
}

template <int NK>
static ScanKernel pick_np(uint32_t np, int kw, bool fast, int sub, bool t3) {
    switch (np) {
        case 0: return pick_kw<NK, 0>(kw, fast, sub, t3);
        case 1: return pick_kw<NK, 1>(kw, fast, sub, t3);
        case 2: return pick_kw<NK, 2>(kw, fast, sub, t3);
        case 3: return pick_kw<NK, 3>(kw, fast, sub, t3);
        default: return pick_kw<NK, 4>(kw, fast, sub, t3);
    }
}

}  // namespace

namespace skb {
// the kernel as an opaque handle (launched with cudaLaunchKernel by scan.cu)
const void *scan_pick_nk1(uint32_t np, int kw, bool fast, int sub, bool t3) { return (const void *)pick_np<1>(np, kw, fast, sub, t3); }
}  // namespace skb
