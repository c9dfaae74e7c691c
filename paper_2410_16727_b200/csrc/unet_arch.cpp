// Parameter table of the BASELINE U-Net, in PSCK blob order (spec.py:UNetArch.param_shapes).
#include "unet_arch.h"

namespace ps {

std::vector<ParamEntry> unet_param_table() {
    std::vector<ParamEntry> t;
    size_t off = 0;
    auto add = [&](const std::string& n, std::vector<int> s) {
        ParamEntry e{n, s, off};
        off += e.numel();
        t.push_back(e);
    };
    auto res = [&](const std::string& n, int ci, int co) {
        add(n + "_c0_w", {co, ci, 5});
        add(n + "_c0_b", {co});
        add(n + "_gn0_g", {co});
        add(n + "_gn0_b", {co});
        add(n + "_c1_w", {co, co, 5});
        add(n + "_c1_b", {co});
        add(n + "_gn1_g", {co});
        add(n + "_gn1_b", {co});
        add(n + "_film_w", {U_FILM_IN, 2 * co});
        add(n + "_film_b", {2 * co});
        if (ci != co) {
            add(n + "_res_w", {co, ci, 1});
            add(n + "_res_b", {co});
        }
    };
    add("t_fc1_w", {U_TEMB, U_THID});
    add("t_fc1_b", {U_THID});
    add("t_fc2_w", {U_THID, U_TEMB});
    add("t_fc2_b", {U_TEMB});
    res("d0r0", U_DOF, 64);
    res("d0r1", 64, 64);
    add("down0_w", {64, 64, 3});
    add("down0_b", {64});
    res("d1r0", 64, 128);
    res("d1r1", 128, 128);
    add("down1_w", {128, 128, 3});
    add("down1_b", {128});
    res("d2r0", 128, 256);
    res("d2r1", 256, 256);
    res("m0", 256, 256);
    res("m1", 256, 256);
    res("u0r0", 512, 128);
    res("u0r1", 128, 128);
    add("up0_w", {128, 128, 4});
    add("up0_b", {128});
    res("u1r0", 256, 64);
    res("u1r1", 64, 64);
    add("up1_w", {64, 64, 4});
    add("up1_b", {64});
    add("fin_c_w", {64, 64, 5});
    add("fin_c_b", {64});
    add("fin_gn_g", {64});
    add("fin_gn_b", {64});
    add("out_w", {U_DOF, 64, 1});
    add("out_b", {U_DOF});
    return t;
}

const ParamEntry* find_param(const std::vector<ParamEntry>& t, const std::string& name) {
    for (const auto& e : t)
        if (e.name == name) return &e;
    return nullptr;
}

}  // namespace ps
