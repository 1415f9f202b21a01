// plan_main.cpp — minimal `hetplan plan` front end over the reference's own
// cli::cmd_plan (tools/cli.cpp:216-260), standing in for tools/main.cpp whose
// CLI11 dependency is not in this image. Linked once with the B200 search
// (integration/Makefile: hetplan_plan_b200) and once with the reference's
// CPU search (hetplan_plan_ref, test infrastructure) so the two CLIs' outputs
// (plan.json, report.json, search_log.ndjson) can be compared byte for byte.
//
//   hetplan_plan --model M --cluster C --train T [--planner P] [--profiles F]
//                [--out DIR] [--jobs N] [--set doc.path=value ...]
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "cli.hpp"

int main(int argc, char** argv) {
  hetplan::cli::Options o;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (i + 1 >= argc) {
      std::cerr << "missing value for " << a << "\n";
      return 64;
    }
    std::string v = argv[++i];
    if (a == "--model") o.model_path = v;
    else if (a == "--cluster") o.cluster_path = v;
    else if (a == "--train") o.train_path = v;
    else if (a == "--planner") o.planner_path = v;
    else if (a == "--profiles") o.profiles_path = v;
    else if (a == "--out") o.out_path = v;
    else if (a == "--jobs") o.jobs = std::atoi(v.c_str());
    else if (a == "--set") o.overrides.push_back(v);
    else {
      std::cerr << "unknown option " << a << "\n";
      return 64;
    }
  }
  return hetplan::cli::cmd_plan(o, std::cout, std::cerr);
}
