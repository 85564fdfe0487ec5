// Product-side TP x PP partition + per-rank arena layout (DESIGN.md §3 / reading #12, #27).
//
// P:138 (§5.1): "Each TP shard still contains the same number of tensors as the
// original model albeit smaller". Megatron 1-D TP split (reading #12): column-parallel
// q/k/v/fc1 (weight rows + bias), row-parallel out_proj/fc2 (weight columns, stored contiguously
// as [out, in/t]; bias replicated), vocab-parallel embed_tokens rows (lm_head tied), replicated
// embed_positions and LayerNorms. PP ("Workers are launched per GPU in accordance with a
// user-provided parallel configuration (TP and PP dimensions)"; reading #27): stage s holds the
// layers [s*L/pp, (s+1)*L/pp); stage 0 also holds embed_tokens + embed_positions; the last
// stage holds the final LayerNorm and, when pp > 1, its own copy of embed_tokens for the tied
// lm_head. Order inside a rank's arena = HF OPTForCausalLM.named_parameters() order restricted
// to the tensors the rank holds; each starts 256-B aligned (one pinned blob per rank).
// tensor_id is the tensor's index in the FULL canonical list (the C0 generator key).
#include "internal.h"

#include <cstdio>
#include <cstring>

namespace mpsw {

static constexpr uint64_t kAlign = 256;

mpsw_status compute_layout(const mpsw_opt_dims& d, int tp, int pp, int stage, int rank, int dtype, Layout& out) {
    if (d.n_layers < 1 || d.hidden < 1 || d.heads < 1 || d.ffn < 1 || d.vocab < 1 || d.max_pos < 1)
        return set_error(MPSW_EINVAL, "dims must be positive");
    if (d.hidden % d.heads) return set_error(MPSW_EINVAL, "hidden % heads != 0");
    if (tp < 1 || d.heads % tp || d.vocab % tp || d.ffn % tp || d.hidden % tp)
        return set_error(MPSW_EINVAL, "tp must divide heads, vocab, ffn and hidden");
    if (pp < 1 || d.n_layers % pp) return set_error(MPSW_EINVAL, "pp must divide n_layers");
    if (stage < 0 || stage >= pp) return set_error(MPSW_EINVAL, "stage out of range");
    if (rank < 0 || rank >= tp) return set_error(MPSW_EINVAL, "rank out of range");
    if (dtype != MPSW_BF16 && dtype != MPSW_FP32) return set_error(MPSW_EINVAL, "bad dtype");
    const uint64_t es = dtype == MPSW_BF16 ? 2 : 4;
    const int h = d.hidden, ff = d.ffn, V = d.vocab, P = d.max_pos + 2;
    const int l0 = stage * (d.n_layers / pp), l1 = (stage + 1) * (d.n_layers / pp);
    const bool first = stage == 0, last = stage == pp - 1;
    out.t.clear();
    uint64_t off = 0;
    int tid = 0;
    auto add = [&](bool hold, const std::string& name, int rows, int cols, int split) {
        const int id = tid++;
        if (!hold) return;
        mpsw_tensor_desc t{};
        std::snprintf(t.name, sizeof(t.name), "%s", name.c_str());
        t.rows = rows;
        t.cols = cols;
        t.split = split;
        t.offset = off;
        t.bytes = (uint64_t)rows * cols * es;
        t.tensor_id = id;
        out.t.push_back(t);
        off = (off + t.bytes + kAlign - 1) / kAlign * kAlign;
    };
    add(first || last, "decoder.embed_tokens.weight", V / tp, h, 1);
    add(first, "decoder.embed_positions.weight", P, h, 0);
    add(last, "decoder.final_layer_norm.weight", h, 1, 0);
    add(last, "decoder.final_layer_norm.bias", h, 1, 0);
    for (int i = 0; i < d.n_layers; ++i) {
        const bool hold = i >= l0 && i < l1;
        const std::string p = "decoder.layers." + std::to_string(i) + ".";
        for (const char* proj : {"k_proj", "v_proj", "q_proj"}) {
            add(hold, p + "self_attn." + proj + ".weight", h / tp, h, 1);
            add(hold, p + "self_attn." + proj + ".bias", h / tp, 1, 1);
        }
        add(hold, p + "self_attn.out_proj.weight", h, h / tp, 2);
        add(hold, p + "self_attn.out_proj.bias", h, 1, 0);
        add(hold, p + "self_attn_layer_norm.weight", h, 1, 0);
        add(hold, p + "self_attn_layer_norm.bias", h, 1, 0);
        add(hold, p + "fc1.weight", ff / tp, h, 1);
        add(hold, p + "fc1.bias", ff / tp, 1, 1);
        add(hold, p + "fc2.weight", h, ff / tp, 2);
        add(hold, p + "fc2.bias", h, 1, 0);
        add(hold, p + "final_layer_norm.weight", h, 1, 0);
        add(hold, p + "final_layer_norm.bias", h, 1, 0);
    }
    out.bytes = off;
    return MPSW_OK;
}

}  // namespace mpsw
