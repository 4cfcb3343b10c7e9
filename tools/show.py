import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], "%.3e" % d["value"], "frac %.3f" % d["roofline"]["frac"], "dag %.3f ms" % d["roofline"]["kernel_ms"],
              "iter %.3f" % d["breakdown_ms"]["pcg_iteration"], "tasks", d["config"].get("dag_tasks"), "setup %.1f" % d["config"].get("setup_seconds", 0))
    except Exception as e:
        print(f, "ERR", e)
