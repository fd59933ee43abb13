// k_tile_bf16.cu — k_doc_score instantiated for bfloat16 sketch cells (SURVEY §8(f) F3,
// DESIGN.md R21): the same kernel (k_doc.cuh) with the column staged as bfloat16 bits and widened
// to fp32 at decode; its own translation unit so that both cell types compile in parallel.
#include "k_doc.cuh"

namespace sinn {

void launch_doc_score_bf16(bool emit, const void* args, bool lower, bool head, cudaStream_t s) {
  launch_doc_score_tpl<true>(emit, *reinterpret_cast<const DocArgs*>(args), lower, head, s);
}

}  // namespace sinn
