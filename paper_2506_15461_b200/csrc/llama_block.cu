// LLaMA-style block (RMSNorm -> QKV -> RoPE -> causal attention -> O ->
// RMSNorm -> SwiGLU MLP), bf16 tcgen05 GEMMs or fp32 parity path.
#include "engine.h"

namespace ckf {

std::unique_ptr<BlockImpl> make_llama_block(Engine*) {
  raise(1, "LLaMA block not built yet");
}

}  // namespace ckf
