// acceptance_b200.cpp — runs the reference's own acceptance criteria
// (tests/acceptance.cpp, compiled from /root/reference unchanged) with the
// reference library linked against the libgsb200 adapter (gsopt_b200.cpp) in
// place of src/rasterizer.cpp: every render / render_backward inside
// estimate_pose, joint_optimize, synth_scene, ... runs on the B200.
//
// The reference's main() runs all nine criteria; this driver selects them by
// number (argv), e.g. `acceptance_b200 2` for criterion 2, pose estimation
// convergence (tests/acceptance.cpp:74-100). Exit code = failures.
#define main gsopt_acceptance_main_unused
#include "acceptance.cpp"
#undef main

#include <cstdlib>

int main(int argc, char** argv) {
  struct Item {
    int id;
    const char* name;
    Outcome (*fn)();
  };
  const Item items[] = {
      {1, "criterion 1: gradient exactness (FD, FP64 tolerance 1e-5)", criterion_gradients},
      {2, "criterion 2: pose estimation convergence (+-15 deg, +-0.15)", criterion_pose_estimation},
      {3, "criterion 3: joint refinement (sigma 0.05 noise, ATE 10x, held-out PSNR)", criterion_joint_refinement},
      {4, "criterion 4: masked relative pose", criterion_masked_relative_pose},
      {5, "criterion 5: Lie-group suite", criterion_lie},
      {6, "criterion 6: loss suite", criterion_losses},
      {7, "criterion 7: pruning contract", criterion_pruning},
      {8, "criterion 8: rendering determinism + performance smoke", criterion_perf},
      {9, "criterion 9: metric suite", criterion_metrics},
  };
  int failures = 0;
  for (int a = 1; a < argc; ++a) {
    const int id = std::atoi(argv[a]);
    for (const Item& it : items)
      if (it.id == id) {
        Outcome o = it.fn();
        std::printf("[%s] %s — %s\n", o.pass ? "PASS" : "FAIL", it.name, o.detail.c_str());
        failures += o.pass ? 0 : 1;
      }
  }
  return failures;
}
