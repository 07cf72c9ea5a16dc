// fast.cu -- XKNN_PREC_BF16 path (tcgen05/TMEM/TMA GEMMs with fused softmax epilogues).
#include "kernels.cuh"

namespace xknn {

xknn_status_t Layer::init_fast() { return XKNN_OK; }
void Layer::free_fast() {}
xknn_status_t Layer::run_fast_core(uint64_t) {
  last_msg = "bf16 path not built yet";
  return XKNN_ERR_UNSUPPORTED;
}

}  // namespace xknn
