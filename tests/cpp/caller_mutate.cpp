// caller_mutate.cpp -- a reference-API client that refills ModelWeights in place between calls.
// The drop-in keeps a device copy per ModelWeights object; it must notice that the values changed.
// Scaling the head by 2 scales every logit by exactly 2 (model.cpp:260-261), in fp64 and in fp32.
#include <cstdio>
#include <vector>

#include "specmoe/model.hpp"

using namespace specmoe;

int main() {
    ModelSpec spec;
    spec.seed = 4;
    ModelWeights w = build_model(spec);
    const std::vector<int> prefix{3, 1, 4, 1, 5};
    ForwardResult a = forward(w, prefix);
    for (double& v : w.head) v *= 2.0;
    ForwardResult b = forward(w, prefix);
    int exact = 1;
    for (size_t i = 0; i < a.logits.size(); ++i) exact &= b.logits[i] == 2.0 * a.logits[i];
    // one mutated expert value must reach the device as well
    w.layers[0].experts[a.activations[0].raw[0]].up[0] += 1.0;
    ForwardResult c = forward(w, prefix);
    int changed = 0;
    for (size_t i = 0; i < b.logits.size(); ++i) changed |= c.logits[i] != b.logits[i];
    std::printf("{\"head_scaled_exact\":%d,\"expert_change_seen\":%d}\n", exact, changed);
    return 0;
}
